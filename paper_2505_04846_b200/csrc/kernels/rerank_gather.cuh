// rerank_gather.cuh -- NEXT N3, stage 2: exact MaxSim of each query against ITS OWN k1 candidates.
//
//   S(q, c) = sum_{i < len_q} max_{j < len_c} < q_i , d_{c,j} >   for c in cand(q)   (§2.2;
//   ColBERTv2's retrieve-then-rerank; SPEC.md:268-276 rerank)
//
// Why a kernel of its own.  Each (query, candidate) pair needs the candidate's token rows and nothing
// else reuses them (candidates of different queries rarely coincide), so the work is a GATHER: one
// chunk's ~len x d bf16 rows (up to 64 KB) per 2 * 32 * len * d FLOP -- 32 FLOP per byte, far below the
// B200 ridge (~250 FLOP/B).  The bound is HBM bandwidth over the gathered rows, not the tensor cores.
// The CTA-pair MaxSim kernel multiplies 8 queries against every chunk it streams, so scoring 8 queries'
// own candidates with it does 8x the necessary MMA work; here every pair is computed exactly once.
//
// Design:
//  * 4 independent warps per CTA, one CTA per SM, each warp owning a contiguous range of the
//    (query, slot) items and its own ring of SW shared-memory stages.  A stage holds one 64-row block of
//    one candidate (all K-blocks, 128B-swizzled TMA boxes of 64 dims x 64 rows); only the chunk's real
//    rows are fetched (ceil(len / 64) blocks), so variable-length chunks cost their own bytes.
//  * Lane 0 issues the TMA for the next blocks as soon as a stage is consumed (up to SW blocks = up to
//    SW * 16 KB in flight per warp); candidate metadata (chunk id, length, first row) for 32 items at
//    a time is prefetched into registers one batch ahead, so no dependent load sits on the issue path.
//  * The query's 32 x d rows stay in registers as mma.sync A fragments for all of its candidates; each
//    64-row block is 2 x 8 x (d/16) mma.sync.m16n8k16 (bf16 -> fp32) with B fragments by ldmatrix from
//    the swizzled stage.  The masked max over the candidate's real rows (R2) is folded in registers
//    per block; the masked sum over the query's real rows (R3) is a fixed butterfly.  The 32 x len
//    similarity tile never leaves registers.
#pragma once
#include <cuda.h>
#include <cuda_bf16.h>
#include <cstdint>

#include "../ptx.cuh"

namespace hiper {

struct RerankArgs {
  const __nv_bfloat16* qlay;  // [n_q_pad][32][dim] NORM'd query rows (hiper_prepare_queries layout)
  const int32_t* q_lens;      // [n_q]
  const int32_t* slots;       // [n_q][k1] local chunk index of each candidate, -1 = not this shard's
  const int32_t* d_lens;      // [n] chunk lengths of the token index
  const int64_t* row_of;      // packed token index: first packed row of chunk c; nullptr = c * ld_pad
  int32_t ld_pad;             // dense token index: rows per chunk
  int32_t dim;
  int32_t k1;
  int64_t n_items;            // n_q * k1
  int64_t n_index;            // chunks in the token index (debug-build bound check)
  float* S2;                  // [n_q][k1] exact MaxSim of each (query, candidate); untouched for -1
};

constexpr int kRerankWarps = 4;

__device__ __forceinline__ void mma_bf16_16816(float (&d)[4], const uint32_t (&a)[4], uint32_t b0,
                                               uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
__device__ __forceinline__ void ldmatrix_x4(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2,
                                            uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// NKB = ceil(dim / 64) (1 or 2); SW = stages per warp.
// tmap64 / tmap16: the token index as 64-dim x 64-row / x 16-row boxes (a chunk's last block is fetched
// in 16-row boxes: only roundup(len, 16) rows ever leave HBM).
template <int NKB, int SW>
__global__ void __launch_bounds__(kRerankWarps * 32, 1)
    rerank_gather_kernel(const __grid_constant__ CUtensorMap tmap64,
                         const __grid_constant__ CUtensorMap tmap16, const RerankArgs a) {
  constexpr uint32_t kStage = 64u * 128u * NKB;  // one 64-row block, all K-blocks
  constexpr int KS = NKB * 4;                    // k16 steps
  extern __shared__ uint8_t smem_raw[];
  using namespace ptx;
  const uint32_t warp = warp_id(), lane = lane_id();
  const uint32_t base = (smem_u32(smem_raw) + 1023u) & ~1023u;
  const uint32_t ring = base + warp * SW * kStage;
  const uint32_t bars = base + kRerankWarps * SW * kStage + warp * SW * 8u;
  if (lane == 0) {
    for (int s = 0; s < SW; ++s) mbar_init(bars + 8u * s, 1);
    fence_mbarrier_init();
  }
  __syncwarp();
  if (warp == 0 && lane == 0) {
    prefetch_tmap(&tmap64);
    prefetch_tmap(&tmap16);
  }

  const int64_t gw = (int64_t)blockIdx.x * kRerankWarps + warp;
  const int64_t nw = (int64_t)gridDim.x * kRerankWarps;
  const int64_t i0 = a.n_items * gw / nw, i1 = a.n_items * (gw + 1) / nw;
  const int64_t n_rel = i1 - i0;
  const uint32_t g = lane >> 2, t4 = lane & 3u;

  // candidate metadata of 32 items (lane j <- item b*32 + j): chunk, length, first row
  auto load_meta = [&](int64_t b, int32_t& mc, int32_t& ml, int64_t& mr) {
    const int64_t rel = b * 32 + lane;
    mc = -1, ml = 0, mr = 0;
    if (rel < n_rel) {
      mc = __ldg(a.slots + i0 + rel);
      HIPER_DASSERT(mc < a.n_index, mc, a.n_index);
      if (mc >= 0) {
        ml = __ldg(a.d_lens + mc);
        mr = a.row_of != nullptr ? __ldg(a.row_of + mc) : (int64_t)mc * a.ld_pad;
      }
    }
  };
  int32_t cur_c, cur_l, nxt_c, nxt_l;
  int64_t cur_r, nxt_r;
  load_meta(0, cur_c, cur_l, cur_r);
  load_meta(1, nxt_c, nxt_l, nxt_r);
  int64_t cb = 0;  // consumer's metadata batch
  auto meta_of = [&](int64_t rel, int32_t& c, int32_t& len, int64_t& row) -> bool {
    const int64_t b = rel >> 5;
    const int j = (int)(rel & 31);
    const bool in_cur = b == cb;
    c = __shfl_sync(0xffffffffu, in_cur ? cur_c : nxt_c, j);
    len = __shfl_sync(0xffffffffu, in_cur ? cur_l : nxt_l, j);
    row = __shfl_sync(0xffffffffu, in_cur ? cur_r : nxt_r, j);
    return b == cb || b == cb + 1;
  };

  // producer cursor (warp-uniform): next item / row block to fetch
  int64_t pit = 0;
  int32_t prb = 0, inflight = 0, s_issue = 0, s_use = 0;
  uint32_t phase = 0;  // bit s: parity of stage s's next completion
  auto pump = [&]() {
    while (inflight < SW && pit < n_rel) {
      int32_t c, len;
      int64_t row;
      if (!meta_of(pit, c, len, row)) break;  // metadata two batches ahead: not loaded yet
      if (c < 0 || prb >= ((len + 63) >> 6)) {
        ++pit;
        prb = 0;
        continue;
      }
      if (lane == 0) {
        const uint32_t bar = bars + 8u * s_issue;
        const uint32_t dst = ring + s_issue * kStage;
        const int32_t r0 = (int32_t)(row + 64 * prb);
        fence_proxy_async_smem();  // the stage's previous ldmatrix reads precede this async write
        const int32_t rows = min(64, len - 64 * prb);
        if (rows == 64) {
          mbar_arrive_expect_tx(bar, kStage);
#pragma unroll
          for (int kb = 0; kb < NKB; ++kb) tma_load_2d(dst + kb * 8192u, &tmap64, bar, kb * 64, r0);
        } else {  // the chunk's last block: roundup(rows, 16) rows in 16-row boxes
          const int32_t n16 = (rows + 15) >> 4;
          mbar_arrive_expect_tx(bar, (uint32_t)n16 * 2048u * NKB);
          for (int32_t b = 0; b < n16; ++b)
#pragma unroll
            for (int kb = 0; kb < NKB; ++kb)
              tma_load_2d(dst + kb * 8192u + (uint32_t)b * 2048u, &tmap16, bar, kb * 64, r0 + 16 * b);
        }
      }
      if (++s_issue == SW) s_issue = 0;
      ++inflight;
      ++prb;
    }
  };

  int32_t cached_q = -1, lq = 0;
  uint32_t af[2][KS][4];  // A fragments of the current query (m16 tiles x k16 steps)
  for (int64_t rel = 0; rel < n_rel; ++rel) {
    if (rel > 0 && (rel & 31) == 0) {  // next metadata batch
      ++cb;
      cur_c = nxt_c, cur_l = nxt_l, cur_r = nxt_r;
      load_meta(cb + 1, nxt_c, nxt_l, nxt_r);
    }
    pump();
    int32_t c, len;
    int64_t row;
    meta_of(rel, c, len, row);
    if (c < 0) continue;
    const int64_t item = i0 + rel;
    const int32_t q = (int32_t)(item / a.k1);
    if (q != cached_q) {
      cached_q = q;
      lq = __ldg(a.q_lens + q);
      const __nv_bfloat16* qb = a.qlay + (int64_t)q * 32 * a.dim;
#pragma unroll
      for (int mt = 0; mt < 2; ++mt)
#pragma unroll
        for (int ks = 0; ks < KS; ++ks) {
          const int col = ks * 16 + 2 * (int)t4;
          const bool ok = ks * 16 < a.dim;
          const __nv_bfloat16* r0 = qb + (int64_t)(mt * 16 + g) * a.dim + col;
          const __nv_bfloat16* r1 = r0 + 8 * a.dim;
          af[mt][ks][0] = ok ? __ldg(reinterpret_cast<const uint32_t*>(r0)) : 0u;
          af[mt][ks][1] = ok ? __ldg(reinterpret_cast<const uint32_t*>(r1)) : 0u;
          af[mt][ks][2] = ok ? __ldg(reinterpret_cast<const uint32_t*>(r0 + 8)) : 0u;
          af[mt][ks][3] = ok ? __ldg(reinterpret_cast<const uint32_t*>(r1 + 8)) : 0u;
        }
    }
    float rmax[2][2] = {{-INFINITY, -INFINITY}, {-INFINITY, -INFINITY}};
    const int32_t nrb = (len + 63) >> 6;
    for (int32_t rb = 0; rb < nrb; ++rb) {
      mbar_wait(bars + 8u * s_use, (phase >> s_use) & 1u);
      phase ^= 1u << s_use;
      const uint32_t st = ring + s_use * kStage;
#pragma unroll 2
      for (int nt = 0; nt < 8; ++nt) {
        float acc[2][4] = {{0.f, 0.f, 0.f, 0.f}, {0.f, 0.f, 0.f, 0.f}};
        const uint32_t r = (uint32_t)(nt * 8) + (lane & 7u);  // this lane's ldmatrix row
#pragma unroll
        for (int ks = 0; ks < KS; ks += 2) {
          const uint32_t kss = (uint32_t)ks + (lane >> 4);
          const uint32_t j = 2u * (kss & 3u) + ((lane >> 3) & 1u);  // 16-byte chunk in the 128-B row
          const uint32_t addr = st + (kss >> 2) * 8192u + r * 128u + ((j ^ (r & 7u)) << 4);
          uint32_t b0, b1, b2, b3;
          ldmatrix_x4(addr, b0, b1, b2, b3);
#pragma unroll
          for (int mt = 0; mt < 2; ++mt) {
            mma_bf16_16816(acc[mt], af[mt][ks], b0, b1);
            mma_bf16_16816(acc[mt], af[mt][ks + 1], b2, b3);
          }
        }
        // columns = candidate rows rb*64 + nt*8 + 2*t4 + {0, 1}; only real rows enter the max (R2)
        const int32_t c0 = rb * 64 + nt * 8 + 2 * (int32_t)t4;
        const bool v0 = c0 < len, v1 = c0 + 1 < len;
#pragma unroll
        for (int mt = 0; mt < 2; ++mt) {
          rmax[mt][0] = fmaxf(rmax[mt][0], fmaxf(v0 ? acc[mt][0] : -INFINITY, v1 ? acc[mt][1] : -INFINITY));
          rmax[mt][1] = fmaxf(rmax[mt][1], fmaxf(v0 ? acc[mt][2] : -INFINITY, v1 ? acc[mt][3] : -INFINITY));
        }
      }
      __syncwarp();  // every lane's ldmatrix of this stage is done: it may be refilled
      if (++s_use == SW) s_use = 0;
      --inflight;
      pump();
    }
    // max over the 4 lanes sharing a query row, then the masked sum over the query's real rows
#pragma unroll
    for (int mt = 0; mt < 2; ++mt)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        rmax[mt][h] = fmaxf(rmax[mt][h], __shfl_xor_sync(0xffffffffu, rmax[mt][h], 1));
        rmax[mt][h] = fmaxf(rmax[mt][h], __shfl_xor_sync(0xffffffffu, rmax[mt][h], 2));
      }
    const int32_t rw = (int32_t)g;  // rows g, g + 8, g + 16, g + 24
    float sv = ((rw < lq ? rmax[0][0] : 0.f) + (rw + 8 < lq ? rmax[0][1] : 0.f)) +
               ((rw + 16 < lq ? rmax[1][0] : 0.f) + (rw + 24 < lq ? rmax[1][1] : 0.f));
#pragma unroll
    for (int o = 4; o <= 16; o <<= 1) sv += __shfl_xor_sync(0xffffffffu, sv, o);
    if (lane == 0) a.S2[item] = sv + 0.0f;
  }
}

}  // namespace hiper
