// peer_gather.cuh -- NEXT N2's cross-rank gather of pooled passages, over NVLink peer memory.
//
// "pooled embeddings from all ranks are gathered, and loss is calculated with the local rank compared
// to min(N, W) samples, where N is the maximum to consider and W is the total samples across all
// ranks" (§3.2.1); the order is the local rank's positives first, then the other ranks'
// rows in (rank, position) order.
//
// Every rank NORMs its b pooled passages into its own WINDOW -- a device buffer exported once with
// CUDA IPC and mapped by every peer (hiper_comm's peer windows) -- and publishes a ready epoch.  This
// kernel builds the m = min(N, W) candidate rows in that order by reading the local window and the
// peers' windows directly over NVLink (16-byte loads, coalesced), after waiting (acquire, system
// scope) until each peer's ready epoch reaches this call's epoch.  It replaces an ncclAllGather into
// a scratch buffer plus world device-to-device reorder copies: one launch, no host round trip, only
// the m rows the loss uses are moved.  Windows alternate by epoch parity, so a rank overwrites the
// buffer of call e only at call e + 2, after every peer has published e + 1 -- i.e. finished reading e.
#pragma once
#include <cuda_bf16.h>
#include <cstdint>

#include "../ptx.cuh"

namespace hiper {

constexpr int kMaxPeers = 64;

struct PeerGatherArgs {
  const __nv_bfloat16* src[kMaxPeers];   // per rank: its NORM'd passages of this epoch, [b][dp]
  const unsigned long long* ready[kMaxPeers];  // per rank: its ready-epoch word (nullptr: no wait)
  unsigned long long epoch;
  int32_t world, rank, b, dp;
  int64_t m;                             // candidate rows to build (<= world * b)
  __nv_bfloat16* cand;                   // [m][dp] out, local HBM
};

__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

// One block per candidate row (grid = m); thread t copies 16-byte word t, t + blockDim, ...
__global__ void __launch_bounds__(128) peer_gather_kernel(const PeerGatherArgs a) {
  const int64_t c = blockIdx.x;
  if (c >= a.m) return;
  // candidate c -> (source rank, row): local first, then the other ranks in rank order
  int32_t r, row;
  if (c < a.b) {
    r = a.rank;
    row = (int32_t)c;
  } else {
    const int64_t o = c - a.b;
    const int32_t k = (int32_t)(o / a.b);
    r = k < a.rank ? k : k + 1;
    row = (int32_t)(o - (int64_t)k * a.b);
  }
  HIPER_DASSERT(r >= 0 && r < a.world && row >= 0 && row < a.b, r, row);
  if (a.ready[r] != nullptr && threadIdx.x == 0) {
    while (ld_acquire_sys(a.ready[r]) < a.epoch) __nanosleep(128);
  }
  __syncthreads();
  const uint4* src = reinterpret_cast<const uint4*>(a.src[r] + (int64_t)row * a.dp);
  uint4* dst = reinterpret_cast<uint4*>(a.cand + c * a.dp);
  for (int32_t w = threadIdx.x; w < a.dp / 8; w += blockDim.x) dst[w] = src[w];
}

// Publish "my passages of `epoch` are in my window" (after the NORM launch, in stream order).
__global__ void peer_signal_kernel(unsigned long long* ready, unsigned long long epoch) {
  __threadfence_system();
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(ready), "l"(epoch) : "memory");
}

}  // namespace hiper
