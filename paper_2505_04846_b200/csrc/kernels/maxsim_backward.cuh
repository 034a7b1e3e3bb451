// maxsim_backward.cuh -- NEXT N1: gradient of the ColTrast late-interaction loss L_LI.
//
// Chain rule (the objective is trained by backpropagation):
//   G_ij          = (softmax_j(S_i / tau)_j - [j == pos_i]) / (B tau)   infonce_rows_kernel (G out)
//   a(i,t,j)      = argmax_{u < len_j} <qn_{i,t}, dn_{j,u}>  (saved by the forward, MODE 2)
//   g_q(i,t)      = sum_j G_ij dn_{j, a(i,t,j)}                  grad_q_stream_kernel + _reduce
//   g_d(j,u)      = sum_i sum_{t: a(i,t,j) = u} G_ij qn_{i,t}       grad_d_sort_kernel + _seg
//   dL/dx (row)   = inv (g - y (y . g)),  y = x inv, inv = 1 / ||x||   (NORM's Jacobian; skipped
//                   with HIPER_ASSUME_NORMALIZED)
// qn / dn are the bf16 NORM'd operands of the forward (the kernels' layouts); the Jacobian uses the
// fp32 y = x * inv of the raw row.  All sums run in a fixed order (deterministic).
#pragma once
#include <cuda.h>
#include <cuda_bf16.h>
#include <cstdint>

#include "../ptx.cuh"

namespace hiper {

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
  ptx::grid_dependency_wait();  // PDL: launched early, waits for its predecessor here
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

// Exclusive prefix sum of one int per thread over an NW-warp block; `total` gets the block sum.
// `wsum` is NW ints of shared memory (reusable once the call returns).
template <int NW>
__device__ __forceinline__ int32_t block_excl_scan(int32_t v, int32_t* wsum, int32_t& total) {
  static_assert(NW <= 32, "one warp scans the warp sums");
  const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int32_t x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int32_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= (uint32_t)o) x += y;
  }
  if (lane == 31) wsum[warp] = x;
  __syncthreads();
  if (warp == 0) {
    int32_t w = lane < (uint32_t)NW ? wsum[lane] : 0;
#pragma unroll
    for (int o = 1; o < NW; o <<= 1) {
      const int32_t y = __shfl_up_sync(0xffffffffu, w, o);
      if (lane >= (uint32_t)o) w += y;
    }
    if (lane < (uint32_t)NW) wsum[lane] = w;
  }
  __syncthreads();
  const int32_t excl = x - v + (warp > 0 ? wsum[warp - 1] : 0);
  total = wsum[NW - 1];
  __syncthreads();
  return excl;
}

// The lanes whose 9-bit key equals this lane's (__match_any_sync's result) from 9 ballots: MATCH.ANY
// has a long latency on this part and sat on the sort's critical path.
__device__ __forceinline__ uint32_t match_any9(int32_t u) {
  uint32_t m = 0xffffffffu;
#pragma unroll
  for (int b = 0; b < 9; ++b) {
    const uint32_t bal = __ballot_sync(0xffffffffu, (u >> b) & 1);
    m &= ((u >> b) & 1) ? bal : ~bal;
  }
  return m;
}

// grad_d, pass 1 -- one block (kSortWarps warps) per doc j: invert the argmax map a(., ., j) with a
// stable counting sort in SMEM:
//  1. stage a(., ., j) (n_q x 32 bytes), G(., j) and q_lens in SMEM;
//  2. warp w histograms its contiguous share of the entries (equal keys per 32 entries by ballots);
//  3. block scans: bucket u of warp w starts at base[u] + sum_{w' < w} hist[w'][u];
//  4. warp w places its entries (stable: lane order within a chunk, chunks in order);
//  5. out: the sorted hits as {i * 32 + t, G_ij} pairs and the bucket starts.
// SMEM: n_q*32*3 + n_q*8 + 2*kSortWarps*257*4 bytes.
constexpr int kSortWarps = 16;
__global__ void __launch_bounds__(kSortWarps * 32) grad_d_sort_kernel(
    const uint8_t* __restrict__ amax, const float* __restrict__ G, int32_t B, int32_t M,
    const int32_t* __restrict__ q_lens, uint2* __restrict__ ent, int32_t* __restrict__ base_out) {
  ptx::grid_dependency_wait();  // PDL: launched early, waits for its predecessor here
  constexpr int NB = 257;  // 256 buckets + 1 for padding entries (t >= len_q)
  constexpr int NW = kSortWarps;
  extern __shared__ uint8_t smem[];
  const int32_t E = B * 32;  // entries (i, t)
  uint8_t* amb = smem;                                                  // [E]
  uint16_t* sorted = reinterpret_cast<uint16_t*>(smem + E);             // [E] entry indices (< 65536)
  float* gcol = reinterpret_cast<float*>(smem + 3 * (size_t)E);         // [B]
  int32_t* lq = reinterpret_cast<int32_t*>(gcol + B);                   // [B]
  int32_t* hist = lq + B;                                               // [NW][NB]
  int32_t* offs = hist + NW * NB;                                       // [NW][NB]
  __shared__ int32_t base[NB + 1];
  __shared__ int32_t wsum[NW];
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
  for (int32_t x = threadIdx.x; x < NW * NB; x += blockDim.x) hist[x] = 0;
  __syncthreads();
  const int32_t per = (E + NW * 32 - 1) / (NW * 32) * 32;  // each warp's range, a multiple of 32
  const int32_t e0 = warp * per;
  auto bucket = [&](int32_t e) -> int32_t {  // entries past E or with t >= len_q go to bucket 256
    return (e < E && (e & 31) < lq[e >> 5]) ? (int32_t)amb[e] : 256;
  };
  for (int32_t c = 0; c < per; c += 32) {
    const int32_t e = e0 + c + lane;
    const int32_t u = bucket(e);
    const uint32_t m = match_any9(u);
    if (lane == (uint32_t)(__ffs(m) - 1)) hist[warp * NB + u] += __popc(m);
    __syncwarp();
  }
  __syncthreads();
  {  // bucket starts: a block scan over buckets 0..255; bucket 256 (padding) goes last
    const int32_t u = threadIdx.x;
    int32_t tot = 0;
    if (u < 256)
#pragma unroll
      for (int32_t w = 0; w < NW; ++w) tot += hist[w * NB + u];
    int32_t all;
    const int32_t ex = block_excl_scan<NW>(tot, wsum, all);
    if (u < 256) base[u] = ex;
    if (u == 0) {
      int32_t pad = 0;
      for (int32_t w = 0; w < NW; ++w) pad += hist[w * NB + 256];
      base[256] = all;
      base[257] = all + pad;
    }
  }
  __syncthreads();
  for (int32_t u = threadIdx.x; u < NB; u += blockDim.x) {
    int32_t run = base[u];
    for (int32_t w = 0; w < NW; ++w) {
      offs[w * NB + u] = run;
      run += hist[w * NB + u];
    }
  }
  __syncthreads();
  for (int32_t c = 0; c < per; c += 32) {
    const int32_t e = e0 + c + lane;
    const int32_t u = bucket(e);
    const uint32_t m = match_any9(u);
    const int32_t rank = __popc(m & ((1u << lane) - 1u));
    if (u < 256) sorted[offs[warp * NB + u] + rank] = (uint16_t)e;
    __syncwarp();
    if (lane == (uint32_t)(__ffs(m) - 1)) offs[warp * NB + u] += __popc(m);
    __syncwarp();
  }
  __syncthreads();
  const int32_t n_hits = base[256];
  for (int32_t x = threadIdx.x; x < n_hits; x += blockDim.x) {
    const uint32_t e = sorted[x];
    ent[(int64_t)j * E + x] = make_uint2(e, __float_as_uint(gcol[e >> 5]));
  }
  for (int32_t x = threadIdx.x; x <= NB; x += blockDim.x) base_out[(int64_t)j * (NB + 1) + x] = base[x];
}

// VPL consecutive values (8- or 16-byte aligned) as floats, one vector load.
template <int VPL>
__device__ __forceinline__ void load_vec(const float* p, float (&x)[VPL]) {
  if constexpr (VPL == 4) {
    const float4 t = *reinterpret_cast<const float4*>(p);
    x[0] = t.x; x[1] = t.y; x[2] = t.z; x[3] = t.w;
  } else {
    const float2 t = *reinterpret_cast<const float2*>(p);
    x[0] = t.x; x[1] = t.y;
  }
}
template <int VPL>
__device__ __forceinline__ void load_vec(const __nv_bfloat16* p, float (&x)[VPL]) {
  if constexpr (VPL == 4) {
    const uint2 t = *reinterpret_cast<const uint2*>(p);
    const float2 a = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&t.x));
    const float2 b = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&t.y));
    x[0] = a.x; x[1] = a.y; x[2] = b.x; x[3] = b.y;
  } else {
    const uint32_t t = *reinterpret_cast<const uint32_t*>(p);
    const float2 a = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&t));
    x[0] = a.x; x[1] = a.y;
  }
}

template <int VPL>
struct RawRow;  // one lane's VPL bf16 values of a row, as raw words
template <>
struct RawRow<4> {
  uint2 w;
  __device__ __forceinline__ void load(const __nv_bfloat16* p) { w = __ldg(reinterpret_cast<const uint2*>(p)); }
  __device__ __forceinline__ void fma(float g, float (&acc)[4]) const {
    const float2 a = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&w.x));
    const float2 b = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&w.y));
    acc[0] = fmaf(g, a.x, acc[0]);
    acc[1] = fmaf(g, a.y, acc[1]);
    acc[2] = fmaf(g, b.x, acc[2]);
    acc[3] = fmaf(g, b.y, acc[3]);
  }
};
template <>
struct RawRow<2> {
  uint32_t w;
  __device__ __forceinline__ void load(const __nv_bfloat16* p) { w = __ldg(reinterpret_cast<const uint32_t*>(p)); }
  __device__ __forceinline__ void fma(float g, float (&acc)[2]) const {
    const float2 a = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&w));
    acc[0] = fmaf(g, a.x, acc[0]);
    acc[1] = fmaf(g, a.y, acc[1]);
  }
};

// grad_d, pass 2 -- one warp per SEGMENT: S consecutive hits of doc j's sorted list (segment s covers
// positions [s S, (s + 1) S)), whatever rows they belong to, so every warp does the same work however
// the hits are spread over rows (a few "hub" doc rows take most of them).  The warp walks its hits 32
// at a time (32 query rows in flight, raw bf16 words) and sums G_ij qn_{i,t} into a running row:
//  * a row that lies inside the segment: its sum g_d(j, u) goes to the output row;
//  * a row that crosses a segment boundary: its partial goes to slot (s, 0) -- the row began before the
//    segment -- or (s, 1) -- it begins in it.
// Pass 3 (grad_d_finish_kernel) adds the partials in segment order and applies NORM's Jacobian, so
// every sum runs in a fixed order (deterministic) and this pass only streams stores.
template <int VPL>
__global__ void __launch_bounds__(256, 2) grad_d_seg_kernel(
    int32_t B, const __nv_bfloat16* __restrict__ qlay, const uint2* __restrict__ ent,
    const int32_t* __restrict__ base, int32_t log2S, int32_t n_seg, float* __restrict__ scratch,
    int32_t d_max_len, float* __restrict__ grad_d) {
  ptx::grid_dependency_wait();  // PDL: launched early, waits for its predecessor here
  constexpr int D = VPL * 32;
  constexpr int NB = 257;
  constexpr int R = 32;  // rows in flight
  __shared__ int32_t sbase[NB + 1];
  const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int32_t bpd = (n_seg + 7) / 8;  // blocks per doc
  const int32_t j = blockIdx.x / bpd;
  const int32_t s = (blockIdx.x - j * bpd) * 8 + (int32_t)warp;
  const int32_t E = B * 32;
  const uint2* ej = ent + (int64_t)j * E;
  const int32_t S = 1 << log2S;
  const int32_t lo = s * S;
  auto load_ent = [&](int32_t x) { return __ldg(ej + min(x, E - 1)); };
  uint2 nxt = load_ent(lo + (int32_t)lane);  // first batch, in flight across the base staging
  for (int32_t x = threadIdx.x; x <= NB; x += blockDim.x) sbase[x] = __ldg(base + (int64_t)j * (NB + 1) + x);
  __syncthreads();
  const int32_t n_hits = sbase[256];
  if (s >= n_seg || lo >= n_hits) return;
  const int32_t hi = min(lo + S, n_hits);
  // the row holding position lo: the last u with sbase[u] <= lo (rows without hits are skipped)
  int32_t u = 0;
  for (int32_t step = 128; step >= 1; step >>= 1)
    if (u + step <= 255 && sbase[u + step] <= lo) u += step;
  int32_t ub = sbase[u + 1];
  float acc[VPL];
#pragma unroll
  for (int v = 0; v < VPL; ++v) acc[v] = 0.0f;
  auto flush = [&]() {
    const int32_t s0 = sbase[u] >> log2S, s1 = (ub - 1) >> log2S;
    float* dst = s0 == s1 ? grad_d + ((int64_t)j * d_max_len + u) * D
                          : scratch + (((int64_t)j * n_seg + s) * 2 + (s > s0 ? 0 : 1)) * D;
    if constexpr (VPL == 4) {
      *reinterpret_cast<float4*>(dst + lane * 4) = make_float4(acc[0], acc[1], acc[2], acc[3]);
    } else {
      *reinterpret_cast<float2*>(dst + lane * 2) = make_float2(acc[0], acc[1]);
    }
#pragma unroll
    for (int v = 0; v < VPL; ++v) acc[v] = 0.0f;
  };
  for (int32_t bl = lo; bl < hi; bl += R) {
    const uint2 my = nxt;
    if (bl + R < hi) nxt = load_ent(bl + R + (int32_t)lane);
    // lanes past the segment load row 0 with weight 0 (an exact +0 term): all R loads issue at once
    const bool real = bl + (int32_t)lane < hi;
    const int32_t e_l = real ? (int32_t)my.x : 0;
    const float g_l = real ? __uint_as_float(my.y) : 0.0f;
    const __nv_bfloat16* ql = qlay + lane * VPL;
    RawRow<VPL> qv[R];
#pragma unroll
    for (int r = 0; r < R; ++r) qv[r].load(ql + __shfl_sync(0xffffffffu, e_l, r) * D);
    // one pass in hit order; a row that ends before hit r is flushed first (warp-uniform branch)
#pragma unroll
    for (int r = 0; r < R; ++r) {
      if (bl + r == ub && bl + r < hi) {
        flush();
        do {
          ++u;
          ub = sbase[u + 1];
        } while (ub <= bl + r);
      }
      qv[r].fma(__shfl_sync(0xffffffffu, g_l, r), acc);
    }
  }
  flush();  // the segment's last row (it ends at hi, or continues past it)
}

// grad_d, pass 3 -- one warp per FR output rows (j, u .. u + FR - 1), their loads issued together:
// g_d(j, u) is 0 (no hit), the row pass 2 wrote (one segment), or the sum of its segments' partials in
// segment order; then NORM's Jacobian.
template <int VPL, typename Tin>
__global__ void __launch_bounds__(256) grad_d_finish_kernel(
    const int32_t* __restrict__ base, int32_t log2S, int32_t n_seg, const float* __restrict__ scratch,
    int32_t M, const Tin* __restrict__ xd, int32_t d_max_len, const int32_t* __restrict__ d_lens,
    uint32_t assume_normalized, float* __restrict__ grad_d) {
  ptx::grid_dependency_wait();  // PDL: launched early, waits for its predecessor here
  constexpr int D = VPL * 32;
  constexpr int NB = 257;
  constexpr int FR = 4;
  const uint32_t lane = threadIdx.x & 31;
  const int32_t wpd = (d_max_len + FR - 1) / FR;  // warps per doc
  const int64_t w = (int64_t)blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
  if (w >= (int64_t)M * wpd) return;
  const int32_t j = (int32_t)(w / wpd), u0 = (int32_t)(w - (int64_t)j * wpd) * FR;
  const int32_t* bj = base + (int64_t)j * (NB + 1);
  const int32_t lj = __ldg(d_lens + j);
  int32_t rs[FR + 1];
#pragma unroll
  for (int k = 0; k <= FR; ++k) rs[k] = __ldg(bj + min(u0 + k, NB));
  // every row's g and x loads issue together (unconditionally: a row without hits reads a stale
  // g it then ignores); the crossing rows' partials follow
  float g[FR][VPL];
  float x[FR][VPL];
#pragma unroll
  for (int k = 0; k < FR; ++k) {
    const int64_t row = (int64_t)j * d_max_len + min(u0 + k, d_max_len - 1);
    load_vec<VPL>(grad_d + row * D + lane * VPL, g[k]);
    if (!assume_normalized) load_vec<VPL>(xd + row * D + lane * VPL, x[k]);
  }
#pragma unroll
  for (int k = 0; k < FR; ++k) {
    if (rs[k + 1] == rs[k]) {
#pragma unroll
      for (int v = 0; v < VPL; ++v) g[k][v] = 0.0f;
      continue;
    }
    const int32_t s0 = rs[k] >> log2S, s1 = (rs[k + 1] - 1) >> log2S;
    if (s0 == s1) continue;
    // partials in segment order, 4 loads in flight (a missing one adds an exact +0)
#pragma unroll
    for (int v = 0; v < VPL; ++v) g[k][v] = 0.0f;
    const float* sl = scratch + (int64_t)j * n_seg * 2 * D + lane * VPL;
    for (int32_t ss = s0; ss <= s1; ss += 4) {
      float pq[4][VPL];
#pragma unroll
      for (int q = 0; q < 4; ++q)
#pragma unroll
        for (int v = 0; v < VPL; ++v)
          pq[q][v] = ss + q <= s1 ? sl[((int64_t)(ss + q) * 2 + (ss + q > s0 ? 0 : 1)) * D + v] : 0.0f;
#pragma unroll
      for (int q = 0; q < 4; ++q)
#pragma unroll
        for (int v = 0; v < VPL; ++v) g[k][v] += pq[q][v];
    }
  }
#pragma unroll
  for (int k = 0; k < FR; ++k) {
    const int32_t u = u0 + k;
    if (u >= d_max_len) break;
    float* out = grad_d + ((int64_t)j * d_max_len + u) * D + lane * VPL;
    if (u >= lj) {  // padding rows: exactly 0 (their raw x may be anything, even 0)
#pragma unroll
      for (int v = 0; v < VPL; ++v) out[v] = 0.0f;
      continue;
    }
    if (assume_normalized) {
#pragma unroll
      for (int v = 0; v < VPL; ++v) out[v] = g[k][v];
      continue;
    }
    float ss = 0.0f;
#pragma unroll
    for (int v = 0; v < VPL; ++v) ss = fmaf(x[k][v], x[k][v], ss);
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
    const float inv = 1.0f / sqrtf(ss);
    float yg = 0.0f;
#pragma unroll
    for (int v = 0; v < VPL; ++v) yg = fmaf(x[k][v] * inv, g[k][v], yg);
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) yg += __shfl_xor_sync(0xffffffffu, yg, o);
#pragma unroll
    for (int v = 0; v < VPL; ++v) out[v] = inv * (g[k][v] - x[k][v] * inv * yg);
  }
}

}  // namespace hiper
