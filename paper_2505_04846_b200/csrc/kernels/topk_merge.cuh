// topk_merge.cuh -- steps a7 (intra-GPU merge of per-partition lists), a8's consumer (merge of the
// all-gathered per-rank lists) and a9 (decode keys -> (score, id)).
//
// Keys are (orderable(score) << 32) | ~id, so "larger key" == "higher score, then lower id"
// (SPEC.md:176, 196 tie rule; R6) and the k largest keys are the exact top-k whatever the
// order the lists are visited in: the merge is deterministic and bitwise independent of the number
// of partitions or ranks (sharding invariance).  Key 0 = empty slot -> (-inf, -1) (R7).
#pragma once
#include <cstdint>

#include "maxsim_sm100.cuh"

namespace hiper {

__device__ __forceinline__ float key_score(uint64_t key) {
  const uint32_t o = (uint32_t)(key >> 32);
  const uint32_t b = (o & 0x80000000u) ? (o & 0x7FFFFFFFu) : ~o;
  return __uint_as_float(b);
}
__device__ __forceinline__ int64_t key_id(uint64_t key) { return (int64_t)(uint32_t)(~(uint32_t)key); }

// One warp per query.  lists: list l of query q starts at lists + l*list_stride + q*q_stride and holds
// k sorted keys.  Writes out_keys[q][k] (if not null) and/or decoded out_scores/out_ids [q][k].
template <int KR>
__global__ void __launch_bounds__(256) topk_merge_kernel(const uint64_t* __restrict__ lists,
                                                         int32_t n_lists, int64_t list_stride,
                                                         int32_t n_q, int64_t q_stride, int32_t k,
                                                         uint64_t* __restrict__ out_keys,
                                                         float* __restrict__ out_scores,
                                                         int64_t* __restrict__ out_ids) {
  const uint32_t lane = threadIdx.x & 31;
  const int32_t q = blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
  if (q >= n_q) return;
  WarpTopK<KR> top;
  top.init();
  for (int32_t l = 0; l < n_lists; ++l) {
    const uint64_t* src = lists + (int64_t)l * list_stride + (int64_t)q * q_stride;
#pragma unroll
    for (int r = 0; r < KR; ++r) {
      const int i = r * 32 + (int)lane;
      const uint64_t cand = (i < k) ? src[i] : 0ull;
      uint32_t mask = __ballot_sync(0xffffffffu, cand > top.thresh);
      while (mask) {
        const int srcl = __ffs(mask) - 1;
        mask &= mask - 1;
        const uint64_t key = __shfl_sync(0xffffffffu, cand, srcl);
        if (key > top.thresh) top.insert(key, k, lane);
      }
    }
  }
#pragma unroll
  for (int r = 0; r < KR; ++r) {
    const int i = r * 32 + (int)lane;
    if (i < k) {
      const uint64_t key = top.v[r];
      const int64_t o = (int64_t)q * k + i;
      if (out_keys) out_keys[o] = key;
      if (out_scores) out_scores[o] = key ? key_score(key) : -INFINITY;
      if (out_ids) out_ids[o] = key ? key_id(key) : -1;
    }
  }
}

}  // namespace hiper
