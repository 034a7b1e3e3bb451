// maxsim_backward.cuh -- NEXT N1: gradient of the ColTrast late-interaction loss L_LI.
//
// Chain rule (the objective is trained by backpropagation):
//   G_ij          = (softmax_j(S_i / tau)_j - [j == pos_i]) / (B tau)            infonce_grad_kernel
//   a(i,t,j)      = argmax_{u < len_j} <qn_{i,t}, dn_{j,u}>  (saved by the forward, MODE 2)
//   g_q(i,t)      = sum_j G_ij dn_{j, a(i,t,j)}                  grad_q_stream_kernel + _reduce
//   g_d(j,u)      = sum_i sum_{t: a(i,t,j) = u} G_ij qn_{i,t}                      grad_d_kernel
//   dL/dx (row)   = inv (g - y (y . g)),  y = x inv, inv = 1 / ||x||   (NORM's Jacobian; skipped
//                   with HIPER_ASSUME_NORMALIZED)
// qn / dn are the bf16 NORM'd operands of the forward (the kernels' layouts); the Jacobian uses the
// fp32 y = x * inv of the raw row.  All sums run in a fixed order (deterministic, no atomics).
#pragma once
#include <cuda.h>
#include <cuda_bf16.h>
#include <cstdint>

#include "../ptx.cuh"

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

// grad_q by streaming: a CTA owns 8 queries (its 8 consumer warps; lane = query token t) and a range of
// chunks; a producer warp TMA-loads each chunk's NORM'd rows (64-dim x ld_pad boxes, 128B swizzle)
// into a 2-stage ring, and every thread adds G_ij * dn_{j, a(i,t,j)} for its own argmax row straight
// from shared memory into 64 * NKB fp32 registers.  Each chunk tile is read from L2 once per 8 queries
// (by TMA) instead of 256 rows gathered per (query, chunk) warp; the swizzle spreads the 32 lanes'
// random rows over the 8 16-byte bank groups.  Partial sums per chunk range go to `part`
// [R][n_q * 32][D]; grad_q_reduce_kernel adds them in range order (deterministic) and applies NORM's
// Jacobian.
constexpr int kGqWarps = 8;
template <int NKB>
__global__ void __launch_bounds__((kGqWarps + 1) * 32, 1)
    grad_q_stream_kernel(const __grid_constant__ CUtensorMap tmap_d, const float* __restrict__ G,
                         const uint8_t* __restrict__ amax, int32_t B, int32_t M, int32_t ld_pad,
                         const int32_t* __restrict__ q_lens, int32_t R, float* __restrict__ part,
                         int32_t NS) {
  constexpr int D = 64 * NKB;
  extern __shared__ uint8_t smem_raw[];
  using namespace ptx;
  const uint32_t warp = warp_id(), lane = lane_id();
  const uint32_t base = (smem_u32(smem_raw) + 1023u) & ~1023u;
  const uint32_t kb_bytes = (uint32_t)ld_pad * 128u;
  const uint32_t stage_bytes = kb_bytes * NKB;
  const uint32_t bars = base + (uint32_t)NS * stage_bytes;  // full[NS], empty[NS]
  if (threadIdx.x == 0) {
    for (int s = 0; s < NS; ++s) {
      mbar_init(bars + 8u * s, 1);
      mbar_init(bars + 8u * (NS + s), kGqWarps);
    }
    fence_mbarrier_init();
  }
  __syncthreads();
  const int32_t qb = blockIdx.x / R, r = blockIdx.x % R;
  const int32_t j0 = (int32_t)((int64_t)r * M / R), j1 = (int32_t)((int64_t)(r + 1) * M / R);
  if (warp == kGqWarps) {  // producer
    if (lane == 0) {
      prefetch_tmap(&tmap_d);
      for (int32_t j = j0; j < j1; ++j) {
        const uint32_t s = (uint32_t)(j - j0) % (uint32_t)NS, ph = ((uint32_t)(j - j0) / (uint32_t)NS) & 1u;
        mbar_wait(bars + 8u * (NS + s), ph ^ 1u);
        mbar_arrive_expect_tx(bars + 8u * s, stage_bytes);
#pragma unroll
        for (int kb = 0; kb < NKB; ++kb)
          tma_load_2d(base + s * stage_bytes + kb * kb_bytes, &tmap_d, bars + 8u * s, kb * 64, j * ld_pad);
      }
    }
    return;
  }
  const int32_t i = qb * kGqWarps + (int32_t)warp;
  const int32_t t = (int32_t)lane;
  const bool valid = i < B && t < q_lens[i < B ? i : 0];
  float acc[D];
#pragma unroll
  for (int v = 0; v < D; ++v) acc[v] = 0.0f;
  // G_ij and a(i, t, j) of the next chunk are loaded one iteration ahead (L2 latency off the loop)
  auto load_gu = [&](int32_t jj, float& gg, uint32_t& uu) {
    gg = (i < B && jj < j1) ? __ldg(G + (int64_t)i * M + jj) : 0.0f;
    uu = (i < B && jj < j1) ? __ldg(amax + ((int64_t)i * M + jj) * 32 + t) : 0u;
  };
  float g_n;
  uint32_t u_n;
  load_gu(j0, g_n, u_n);
  for (int32_t j = j0; j < j1; ++j) {
    const uint32_t s = (uint32_t)(j - j0) % (uint32_t)NS, ph = ((uint32_t)(j - j0) / (uint32_t)NS) & 1u;
    const float g = g_n;
    const uint32_t u = u_n;
    load_gu(j + 1, g_n, u_n);
    mbar_wait(bars + 8u * s, ph);
    if (valid) {
      const uint32_t row = base + s * stage_bytes + u * 128u;
#pragma unroll
      for (int c = 0; c < 8 * NKB; ++c) {
        const uint32_t addr = row + (uint32_t)(c >> 3) * kb_bytes + ((((uint32_t)c & 7u) ^ (u & 7u)) << 4);
        uint32_t w0, w1, w2, w3;
        asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(w0), "=r"(w1), "=r"(w2), "=r"(w3) : "r"(addr));
        const uint32_t w[4] = {w0, w1, w2, w3};
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          acc[c * 8 + 2 * e] = fmaf(g, __uint_as_float(w[e] << 16), acc[c * 8 + 2 * e]);
          acc[c * 8 + 2 * e + 1] = fmaf(g, __uint_as_float(w[e] & 0xFFFF0000u), acc[c * 8 + 2 * e + 1]);
        }
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(bars + 8u * (NS + s));
  }
  if (i < B) {
    float4* dst = reinterpret_cast<float4*>(part + (((int64_t)r * B + i) * 32 + t) * D);
#pragma unroll
    for (int v = 0; v < D / 4; ++v) dst[v] = make_float4(acc[4 * v], acc[4 * v + 1], acc[4 * v + 2], acc[4 * v + 3]);
  }
}

// One warp per (query i, token t): sum the R partial rows in range order, NORM's Jacobian.
template <int VPL, typename Tin>
__global__ void __launch_bounds__(256) grad_q_reduce_kernel(const float* __restrict__ part, int32_t R,
                                                            int32_t B, const Tin* __restrict__ xq,
                                                            int32_t q_max_len,
                                                            const int32_t* __restrict__ q_lens,
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
  for (int32_t r = 0; r < R; ++r) {
    const float* pr = part + (((int64_t)r * B + i) * 32 + t) * D + lane * VPL;
#pragma unroll
    for (int v = 0; v < VPL; ++v) g[v] += pr[v];
  }
  norm_backward_row<VPL, Tin>(xq + row * D, g, assume_normalized != 0, out, lane);
}

// One block (8 warps) per doc j: invert the argmax map with a stable counting sort in SMEM, then
// gather-sum each output row in (i, t) order.  With sorted_out / base_out set the block only sorts
// and stores the inverted map; grad_d_gather_kernel then runs one warp per output row.
//  1. stage a(., ., j) (n_q x 32 bytes), G(., j) and q_lens in SMEM;
//  2. warp w histograms its contiguous eighth of the entries (match_any per 32 entries);
//  3. block-wide offsets: bucket u of warp w starts at base[u] + sum_{w' < w} hist[w'][u];
//  4. warp w places its entries (stable: lane order within a chunk, chunks in order);
//  5. warp w owns rows u = w, w+8, ...: sum G_ij qn_{i,t} over the bucket (8 gathers in flight, in
//     sorted = (i, t) order: deterministic, no atomics), then NORM's Jacobian.
// SMEM: n_q*32 (argmax) + n_q*32*2 (sorted entries) + n_q*8 + 8*257*4*2 bytes (n_q <= 2048).
template <int VPL, typename Tin>
__global__ void __launch_bounds__(256) grad_d_kernel(const float* __restrict__ G,
                                                     const uint8_t* __restrict__ amax, int32_t B,
                                                     int32_t M, const __nv_bfloat16* __restrict__ qlay,
                                                     const int32_t* __restrict__ q_lens,
                                                     int32_t ld_pad, const Tin* __restrict__ xd,
                                                     int32_t d_max_len, const int32_t* __restrict__ d_lens,
                                                     uint32_t assume_normalized,
                                                     float* __restrict__ grad_d,
                                                     uint16_t* __restrict__ sorted_out = nullptr,
                                                     int32_t* __restrict__ base_out = nullptr) {
  constexpr int D = VPL * 32;
  constexpr int NB = 257;  // 256 buckets + 1 for padding entries (t >= len_q)
  extern __shared__ uint8_t smem[];
  const int32_t E = B * 32;  // entries (i, t)
  uint8_t* amb = smem;                                                  // [E]
  uint16_t* sorted = reinterpret_cast<uint16_t*>(smem + E);             // [E] entry indices (< 65536)
  float* gcol = reinterpret_cast<float*>(smem + 3 * (size_t)E);         // [B]
  int32_t* lq = reinterpret_cast<int32_t*>(gcol + B);                   // [B]
  int32_t* hist = lq + B;                                               // [8][NB]
  int32_t* offs = hist + 8 * NB;                                        // [8][NB]
  __shared__ int32_t base[NB + 1];
  const int32_t j = blockIdx.x;
  const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int32_t w = threadIdx.x; w < E / 4; w += blockDim.x) {
    const int32_t i = w >> 3, k = w & 7;
    reinterpret_cast<uint32_t*>(amb)[w] =
        *reinterpret_cast<const uint32_t*>(amax + ((int64_t)i * M + j) * 32 + k * 4);
  }
  for (int32_t i = threadIdx.x; i < B; i += blockDim.x) {
    gcol[i] = G[(int64_t)i * M + j];
    lq[i] = q_lens[i];
  }
  for (int32_t x = threadIdx.x; x < 8 * NB; x += blockDim.x) hist[x] = 0;
  __syncthreads();
  const int32_t per = (E + 8 * 32 - 1) / (8 * 32) * 32;  // each warp's range, a multiple of 32
  const int32_t e0 = warp * per;
  auto bucket = [&](int32_t e) -> int32_t {  // entries past E or with t >= len_q go to bucket 256
    return (e < E && (e & 31) < lq[e >> 5]) ? (int32_t)amb[e] : 256;
  };
  for (int32_t c = 0; c < per; c += 32) {
    const int32_t e = e0 + c + lane;
    const int32_t u = bucket(e);
    const uint32_t m = __match_any_sync(0xffffffffu, u);
    if (lane == (uint32_t)(__ffs(m) - 1)) hist[warp * NB + u] += __popc(m);
    __syncwarp();
  }
  __syncthreads();
  if (threadIdx.x == 0) {  // exclusive scan over buckets of the per-bucket totals (257 adds)
    int32_t run = 0;
    for (int32_t u = 0; u < NB; ++u) {
      base[u] = run;
      for (int32_t w = 0; w < 8; ++w) run += hist[w * NB + u];
    }
    base[NB] = run;
  }
  __syncthreads();
  for (int32_t u = threadIdx.x; u < NB; u += blockDim.x) {
    int32_t run = base[u];
    for (int32_t w = 0; w < 8; ++w) {
      offs[w * NB + u] = run;
      run += hist[w * NB + u];
    }
  }
  __syncthreads();
  for (int32_t c = 0; c < per; c += 32) {
    const int32_t e = e0 + c + lane;
    const int32_t u = bucket(e);
    const uint32_t m = __match_any_sync(0xffffffffu, u);
    const int32_t rank = __popc(m & ((1u << lane) - 1u));
    if (u < 256) sorted[offs[warp * NB + u] + rank] = (uint16_t)e;
    __syncwarp();
    if (lane == (uint32_t)(__ffs(m) - 1)) offs[warp * NB + u] += __popc(m);
    __syncwarp();
  }
  __syncthreads();
  const int32_t lj = d_lens[j];
  if (sorted_out != nullptr) {  // sort-only mode: hand the inverted map to grad_d_gather_kernel
    for (int32_t x = threadIdx.x; x < E; x += blockDim.x) sorted_out[(int64_t)j * E + x] = sorted[x];
    for (int32_t x = threadIdx.x; x <= NB; x += blockDim.x) base_out[(int64_t)j * (NB + 1) + x] = base[x];
    return;
  }
  for (int32_t u = warp; u < d_max_len; u += 8) {
    float* out = grad_d + ((int64_t)j * d_max_len + u) * D;
    if (u >= lj) {
#pragma unroll
      for (int v = 0; v < VPL; ++v) out[lane * VPL + v] = 0.0f;
      continue;
    }
    float g[VPL];
#pragma unroll
    for (int v = 0; v < VPL; ++v) g[v] = 0.0f;
    const int32_t h0 = base[u], h1 = base[u + 1];
    int32_t h = h0;
    for (; h + 8 <= h1; h += 8) {
      float qv[8][VPL];
      float gv[8];
#pragma unroll
      for (int r = 0; r < 8; ++r) {
        const int32_t e = sorted[h + r];
        gv[r] = gcol[e >> 5];
        const __nv_bfloat16* qr = qlay + (int64_t)e * D + lane * VPL;
#pragma unroll
        for (int v = 0; v < VPL; ++v) qv[r][v] = __bfloat162float(qr[v]);
      }
#pragma unroll
      for (int r = 0; r < 8; ++r)
#pragma unroll
        for (int v = 0; v < VPL; ++v) g[v] = fmaf(gv[r], qv[r][v], g[v]);
    }
    for (; h < h1; ++h) {
      const int32_t e = sorted[h];
      const float gij = gcol[e >> 5];
      const __nv_bfloat16* qr = qlay + (int64_t)e * D + lane * VPL;
#pragma unroll
      for (int v = 0; v < VPL; ++v) g[v] = fmaf(gij, __bfloat162float(qr[v]), g[v]);
    }
    norm_backward_row<VPL, Tin>(xd + ((int64_t)j * d_max_len + u) * D, g, assume_normalized != 0,
                                out, lane);
  }
}

// One warp per doc output row (j, u): gather-sum G_ij qn_{i,t} over the row's bucket of the inverted
// argmax map (sorted (i, t) order from grad_d_kernel's sort-only mode: deterministic), 16 gathers in
// flight, then NORM's Jacobian.  65,536 warps at B = 256 instead of 256 blocks.
template <int VPL, typename Tin>
__global__ void __launch_bounds__(256) grad_d_gather_kernel(const float* __restrict__ G, int32_t B,
                                                            int32_t M, const __nv_bfloat16* __restrict__ qlay,
                                                            const uint16_t* __restrict__ sorted,
                                                            const int32_t* __restrict__ base,
                                                            const Tin* __restrict__ xd, int32_t d_max_len,
                                                            const int32_t* __restrict__ d_lens,
                                                            uint32_t assume_normalized,
                                                            float* __restrict__ grad_d) {
  constexpr int D = VPL * 32;
  constexpr int NB = 257;
  const uint32_t lane = threadIdx.x & 31;
  const int64_t row = (int64_t)blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
  if (row >= (int64_t)M * d_max_len) return;
  const int32_t j = (int32_t)(row / d_max_len), u = (int32_t)(row % d_max_len);
  float* out = grad_d + row * D;
  if (u >= d_lens[j]) {
#pragma unroll
    for (int v = 0; v < VPL; ++v) out[lane * VPL + v] = 0.0f;
    return;
  }
  const int32_t E = B * 32;
  const uint16_t* srt = sorted + (int64_t)j * E;
  const int32_t h0 = base[(int64_t)j * (NB + 1) + u], h1 = base[(int64_t)j * (NB + 1) + u + 1];
  float g[VPL];
#pragma unroll
  for (int v = 0; v < VPL; ++v) g[v] = 0.0f;
  int32_t h = h0;
  for (; h + 16 <= h1; h += 16) {
    float qv[16][VPL];
    float gv[16];
#pragma unroll
    for (int r = 0; r < 16; ++r) {
      const int32_t e = srt[h + r];
      gv[r] = G[(int64_t)(e >> 5) * M + j];
      const __nv_bfloat16* qr = qlay + (int64_t)e * D + lane * VPL;
#pragma unroll
      for (int v = 0; v < VPL; ++v) qv[r][v] = __bfloat162float(qr[v]);
    }
#pragma unroll
    for (int r = 0; r < 16; ++r)
#pragma unroll
      for (int v = 0; v < VPL; ++v) g[v] = fmaf(gv[r], qv[r][v], g[v]);
  }
  for (; h < h1; ++h) {
    const int32_t e = srt[h];
    const float gij = G[(int64_t)(e >> 5) * M + j];
    const __nv_bfloat16* qr = qlay + (int64_t)e * D + lane * VPL;
#pragma unroll
    for (int v = 0; v < VPL; ++v) g[v] = fmaf(gij, __bfloat162float(qr[v]), g[v]);
  }
  norm_backward_row<VPL, Tin>(xd + row * D, g, assume_normalized != 0, out, lane);
}

}  // namespace hiper
