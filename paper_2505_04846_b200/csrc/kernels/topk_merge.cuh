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
// list_len keys (any order; key 0 = empty).  Writes the k largest as out_keys[q][k] (if not null)
// and/or decoded out_scores/out_ids [q][k].
template <int KR>
__global__ void __launch_bounds__(256) topk_merge_kernel(const uint64_t* __restrict__ lists,
                                                         int32_t n_lists, int64_t list_stride,
                                                         int32_t n_q, int64_t q_stride, int32_t k,
                                                         uint64_t* __restrict__ out_keys,
                                                         float* __restrict__ out_scores,
                                                         int64_t* __restrict__ out_ids,
                                                         int32_t list_len) {
  const uint32_t lane = threadIdx.x & 31;
  const int32_t q = blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
  if (q >= n_q) return;
  WarpTopK<KR> top;
  top.init();
  // 8 lists per step: their loads are all in flight before the first is consumed (the banded top-k
  // path produces ~2,000 lists per query at config 3)
  constexpr int U = 8;
  for (int32_t l0 = 0; l0 < n_lists; l0 += U) {
    uint64_t cand[U][KR];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint64_t* src = lists + (int64_t)(l0 + u) * list_stride + (int64_t)q * q_stride;
#pragma unroll
      for (int r = 0; r < KR; ++r) {
        const int i = r * 32 + (int)lane;
        cand[u][r] = (l0 + u < n_lists && i < list_len) ? __ldcs(src + i) : 0ull;
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
#pragma unroll
      for (int r = 0; r < KR; ++r) {
        uint32_t mask = __ballot_sync(0xffffffffu, cand[u][r] > top.thresh);
        while (mask) {
          const int srcl = __ffs(mask) - 1;
          mask &= mask - 1;
          const uint64_t key = __shfl_sync(0xffffffffu, cand[u][r], srcl);
          if (key > top.thresh) top.insert(key, k, lane);
        }
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

// Pooled top-k, APPEND path (16 < k <= 128): query q's n_seg candidate segments (one per (partition,
// group) unit thread: cand[q * n_seg + s][0 .. min(cnt, cap))) hold every corpus key >= its sample
// bound, hence its whole top-k; one warp per query takes the k largest, lane l walking segment l
// of each group of 32.  A segment
// that overflowed (cnt > cap) sets bit 4 of *status (the host then reruns the batch on the heap path).
template <int KR>
__global__ void __launch_bounds__(256) cand_select_kernel(const uint64_t* __restrict__ cand,
                                                          const uint32_t* __restrict__ cnt, int32_t n_seg,
                                                          int32_t cap, int32_t n_q, int32_t k,
                                                          uint64_t* __restrict__ out_keys,
                                                          float* __restrict__ out_scores,
                                                          int64_t* __restrict__ out_ids,
                                                          uint32_t* __restrict__ status) {
  const uint32_t lane = threadIdx.x & 31;
  const int32_t q = blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
  if (q >= n_q) return;
  WarpTopK<KR> top;
  top.init();
  bool over = false;
  // 32 segments at a time, lane l walking segment s0 + l: 4 independent loads per lane per round
  for (int32_t s0 = 0; s0 < n_seg; s0 += 32) {
    const bool live = s0 + (int32_t)lane < n_seg;
    const uint32_t my_c = live ? __ldg(cnt + (int64_t)q * n_seg + s0 + lane) : 0u;
    over |= my_c > (uint32_t)cap;
    const int32_t my_n = (int32_t)min(my_c, (uint32_t)cap);
    int32_t mx = my_n;
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    const uint64_t* src = cand + ((int64_t)q * n_seg + s0 + (live ? (int32_t)lane : 0)) * cap;
    constexpr int U = 4;
    for (int32_t i0 = 0; i0 < mx; i0 += U) {
      uint64_t cv[U];
#pragma unroll
      for (int u = 0; u < U; ++u) cv[u] = i0 + u < my_n ? __ldcs(src + i0 + u) : 0ull;
#pragma unroll
      for (int u = 0; u < U; ++u) {
        uint32_t mask = __ballot_sync(0xffffffffu, cv[u] > top.thresh);
        while (mask) {
          const int srcl = __ffs(mask) - 1;
          mask &= mask - 1;
          const uint64_t key = __shfl_sync(0xffffffffu, cv[u], srcl);
          if (key > top.thresh) top.insert(key, k, lane);
        }
      }
    }
  }
  if (__any_sync(0xffffffffu, over) && lane == 0) atomicOr(status, 16u);
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

// NEXT N3, stage-2 selection: query q's re-scored candidates S[q][0..K1) (slot s valid iff
// cand[q][s] >= 0) -> its exact top-k (score desc, id asc), decoded and/or as keys.  One warp per
// query, K1 <= 128 (32 candidates per round).
template <int KR>
__global__ void __launch_bounds__(256) rerank_select_kernel(const float* __restrict__ S,
                                                            const int32_t* __restrict__ cand,
                                                            int32_t K1, int32_t n_q, int64_t id_base,
                                                            int32_t k, float* __restrict__ out_scores,
                                                            int64_t* __restrict__ out_ids,
                                                            uint64_t* __restrict__ out_keys = nullptr) {
  const uint32_t lane = threadIdx.x & 31;
  const int32_t q = blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
  if (q >= n_q) return;
  WarpTopK<KR> top;
  top.init();
  for (int32_t s0 = 0; s0 < K1; s0 += 32) {
    const int32_t s = s0 + (int32_t)lane;
    uint64_t cand_key = 0ull;
    if (s < K1) {
      const int32_t c = cand[(int64_t)q * K1 + s];
      if (c >= 0) cand_key = make_key(S[(int64_t)q * K1 + s] + 0.0f, id_base + c);
    }
    uint32_t mask = __ballot_sync(0xffffffffu, cand_key > top.thresh);
    while (mask) {
      const int src = __ffs(mask) - 1;
      mask &= mask - 1;
      const uint64_t key = __shfl_sync(0xffffffffu, cand_key, src);
      if (key > top.thresh) top.insert(key, k, lane);
    }
  }
#pragma unroll
  for (int r = 0; r < KR; ++r) {
    const int i = r * 32 + (int)lane;
    if (i < k) {
      const uint64_t key = top.v[r];
      if (out_keys) out_keys[(int64_t)q * k + i] = key;
      if (out_scores) out_scores[(int64_t)q * k + i] = key ? key_score(key) : -INFINITY;
      if (out_ids) out_ids[(int64_t)q * k + i] = key ? key_id(key) : -1;
    }
  }
}

// Stage-1 ids (int64 global, -1 = none) [n_q][K1] -> stage-2 slot table [n_q][K1] of local chunk
// indices; ids outside this shard [id_base, id_base + n) (re-scored by the rank that owns them) -> -1.
__global__ void ids_to_slots_kernel(const int64_t* __restrict__ ids, int64_t n_items, int64_t id_base,
                                    int64_t n, int32_t* __restrict__ slots) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= n_items) return;
  const int64_t id = ids[e];
  HIPER_DASSERT(id >= -1, (uint32_t)id, (uint32_t)e);
  slots[e] = (id >= id_base && id < id_base + n) ? (int32_t)(id - id_base) : -1;
}

}  // namespace hiper
