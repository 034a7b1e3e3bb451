// maxsim_sm100_ts.cuh -- steps a3-a6 with the query tile resident in TENSOR memory (the "TS" form of
// tcgen05.mma: A from TMEM, B from shared memory) and a ring of 7 accumulator slots of 64 columns.
//
//   S(q, c) = sum_{i < len_q} max_{j < len_c} < q_i , d_{c,j} >       (§2.2, Fig.3B
//                                                                    PAPER.md:228)
//
// Why ("Where the cycles go"): in the SS kernel (maxsim_sm100_pair.cuh) a chunk is one
// N = 256 MMA into one of two 256-column accumulators, so the MMA of chunk t+2 can start only after
// the epilogue has drained chunk t -- a round trip (commit -> epilogue wake -> drain -> cluster arrive
// -> MMA wake) measured at ~1,300-1,500 cycles against 1,024 cycles of queued MMA work (the other
// accumulator).  Smaller accumulators would queue more work, but with A in shared memory an N < 256
// MMA re-reads the 4 KB A slab per instruction and saturates the SMEM port.  Here A (this CTA's 128
// query rows x 128 dims) is copied ONCE per unit into TMEM columns [448, 512) (tcgen05.cp from the
// TMA-loaded SMEM tile), every MMA reads it from there, and the remaining 448 columns form 7 slots of
// 64: a chunk is 4 MMAs of N = 64 (its 256 token rows), each into the next slot of the ring, so a slot
// is rewritten only after 6 other slots' work (1,536 MMA cycles) -- and SMEM serves only B (64 B/clk).
//
// Scope: the production shape only -- dense layout, chunk rows ld_pad = 256, dim = 128, queries of
// <= 32 tokens; MODE 1 (per-unit top-k) and MODE 0 (dense scores).  Everything else keeps the SS
// kernel.  Column n of a 64-wide slot j of a chunk is chunk row 32j + n (n < 32, CTA 0's rows) or
// 128 + 32j + (n - 32) (CTA 1's rows): the pair MMA takes the first N/2 B rows from CTA 0's shared
// memory and the rest from CTA 1's, at the same offset.
#pragma once
#include "maxsim_sm100_pair.cuh"

namespace hiper {

constexpr uint32_t kTsACol = 448;

// SN: accumulator slot width = MMA N (64: 7 slots, 4 MMAs per chunk; 128: 3 slots, 2 per chunk).
template <int MODE, int KR, bool STATS = false, int SN = 64>
__global__ void __launch_bounds__(kMaxsimThreads, 1)
    maxsim_ts_kernel(const __grid_constant__ CUtensorMap tmap_q, const __grid_constant__ CUtensorMap tmap_d,
                     const MaxsimArgs args) {
  static_assert(MODE == 0 || MODE == 1, "TS kernel: dense scores or top-k");
  constexpr uint32_t kTsSlotCols = SN, kTsSlots = 448 / SN, kSub = 256 / SN, kHalf = SN / 2;
  extern __shared__ uint8_t smem_raw[];
  using namespace ptx;
  const uint32_t warp = warp_id();
  const uint32_t lane = lane_id();
  const uint32_t rank = cluster_ctarank();  // 0 = leader
  const uint32_t pair = cluster_id_x();
  const uint32_t n_pairs = nclusters_x();

  const uint32_t base = (smem_u32(smem_raw) + 1023u) & ~1023u;
  const uint32_t sA = base;                            // 2 x a_bytes (TMA staging of the A tile)
  const uint32_t sB = sA + 2 * args.a_bytes;           // n_stages x stage_bytes
  const uint32_t sBar = sB + args.n_stages * args.stage_bytes;
  const int S = args.n_stages;
  auto bar_full = [&](int s) { return sBar + 8u * s; };
  auto bar_empty = [&](int s) { return sBar + 8u * (S + s); };
  auto bar_afull = [&](int b) { return sBar + 8u * (2 * S + b); };
  auto bar_aempty = [&](int b) { return sBar + 8u * (2 * S + 2 + b); };
  auto bar_tempty = [&](uint32_t j) { return sBar + 8u * (2 * S + 4 + j); };               // [<= 7]
  auto bar_tfull = [&](uint32_t j, uint32_t g) { return sBar + 8u * (2 * S + 11 + 2 * j + g); };  // [7][2]
  const uint32_t bar_afree = sBar + 8u * (2 * S + 25);  // previous unit's MMAs done with A in TMEM
  const uint32_t sTmemPtr = sBar + 8u * (2 * S + 26);
  uint32_t* tmem_ptr_generic = reinterpret_cast<uint32_t*>(smem_raw + (sTmemPtr - smem_u32(smem_raw)));

  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(bar_full(s), 1);
      mbar_init(bar_empty(s), 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(bar_afull(b), 1);
      mbar_init(bar_aempty(b), 1);
    }
    for (uint32_t j = 0; j < kTsSlots; ++j) {
      mbar_init(bar_tempty(j), 8);  // 4 warps of the draining group in each of the 2 CTAs
      mbar_init(bar_tfull(j, 0), 1);
      mbar_init(bar_tfull(j, 1), 1);
    }
    mbar_init(bar_afree, 1);
    fence_mbarrier_init();
  }
  if (warp == kPairAllocWarp) {
    tmem_alloc_pair(sTmemPtr, kTmemCols);
    tmem_relinquish_pair();
  }
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem_base = *reinterpret_cast<volatile uint32_t*>(tmem_ptr_generic);
  grid_dependency_wait();

  const int32_t n_units = args.n_groups * args.n_parts;
  const uint32_t half_tile = 128u * 128u;  // one 64-dim K-block of this CTA's 128 chunk rows
  long long st_drain = 0, st_ewait = 0, st_tiles = 0;  // STATS (epilogue warps)

  if (warp == kPairProducerWarp) {
    // ================= TMA producer (both CTAs): as the SS kernel =================
    if (lane == 0) {
      prefetch_tmap(&tmap_q);
      prefetch_tmap(&tmap_d);
    }
    int s = 0;
    uint32_t ph = 0, it = 0, streamed = 0;
    for (int32_t u = (int32_t)pair; u < n_units; u += (int32_t)n_pairs, ++it) {
      int32_t g, p;
      int64_t c0, c1;
      unit_decode(args, u, g, p, c0, c1);
      if (lane == 0) {
        const uint32_t ab = it & 1u, aph = (it >> 1) & 1u;
        mbar_wait(bar_aempty(ab), aph ^ 1u);
        if (rank == 0) mbar_arrive_expect_tx(bar_afull(ab), 2u * args.a_bytes);
        const uint32_t afull_leader = mapa_shared(bar_afull(ab), 0);
        for (int kb = 0; kb < 2; ++kb)
          tma_load_2d_pair(sA + ab * args.a_bytes + kb * 16384u, &tmap_q, afull_leader, kb * 64,
                           (int32_t)((2 * g + (int32_t)rank) * 128));
        for (int64_t c = c0; c < c1; ++c) {
          if (args.progress != nullptr && rank == 0 && ((c - c0) & 15) == 0) {
            const uint32_t pos = streamed + (uint32_t)(c - c0);
            lockstep_publish(args.progress, pair, pos);
            lockstep_wait(args.progress, n_pairs, pos, (uint32_t)args.window);
          }
          mbar_wait(bar_empty(s), ph ^ 1u);
          if (rank == 0) mbar_arrive_expect_tx(bar_full(s), 2u * args.stage_bytes);
          const uint32_t full_leader = mapa_shared(bar_full(s), 0);
          const int32_t brow = (int32_t)(c * 256 + (int64_t)rank * 128);
          for (int kb = 0; kb < 2; ++kb)
            tma_load_2d_pair(sB + s * args.stage_bytes + kb * half_tile, &tmap_d, full_leader, kb * 64, brow);
          if (++s == S) { s = 0; ph ^= 1u; }
        }
      }
      __syncwarp();
      streamed += (uint32_t)(c1 - c0);
    }
    if (lane == 0 && args.progress != nullptr && rank == 0) lockstep_publish(args.progress, pair, 0xFFFFFFFFu);
  } else if (warp == kPairMmaWarp) {
    // ================= MMA issuer: leader CTA, single thread =================
    if (rank == 0 && lane == 0) {
      const uint32_t idesc = idesc_bf16_f32(256, kTsSlotCols);
      const uint32_t a_tmem = tmem_base + kTsACol;
      int s = 0;
      uint32_t ph = 0, it = 0, slot = 0;
      uint32_t empty_ph = 0;  // bit j: parity of slot j's next use
      uint32_t tmsb = 0;      // chunk counter parity source for the draining group
      long long st_acc = 0, st_full = 0, st_issue = 0;
      const long long st_t0 = clock64();
      for (int32_t u = (int32_t)pair; u < n_units; u += (int32_t)n_pairs, ++it) {
        int32_t g, p;
        int64_t c0, c1;
        unit_decode(args, u, g, p, c0, c1);
        const uint32_t ab = it & 1u, aph = (it >> 1) & 1u;
        mbar_wait(bar_afull(ab), aph);
        if (it > 0) mbar_wait(bar_afree, (it - 1) & 1u);  // the last unit's MMAs no longer read A
        tc_fence_after();
        // A -> TMEM: 8 K-steps of 16 (128 rows x 256 bits each), both CTAs
#pragma unroll
        for (int ks = 0; ks < 8; ++ks)
          tmem_cp_128x256b_pair(a_tmem + 8u * ks,
                                umma_desc_sw128(sA + ab * args.a_bytes + (ks >> 2) * 16384u + (ks & 3) * 32));
        mma_commit_pair_mc(bar_aempty(ab), 0x3);  // the SMEM A tile is free once the copies land
        for (int64_t c = c0; c < c1; ++c, ++tmsb) {
          const uint32_t grp = tmsb & 1u;
          long long w0 = STATS ? clock64() : 0;
          mbar_wait(bar_full(s), ph);
          if (STATS) st_full += clock64() - w0;
          tc_fence_after();
          const uint32_t b_st = sB + s * args.stage_bytes;
#pragma unroll 1
          for (uint32_t j = 0; j < kSub; ++j) {
            long long w1 = STATS ? clock64() : 0;
            mbar_wait(bar_tempty(slot), ((empty_ph >> slot) & 1u) ^ 1u);
            empty_ph ^= 1u << slot;
            if (STATS) {
              st_acc += clock64() - w1;
              w1 = clock64();
            }
            tc_fence_after();
            const uint32_t d_tmem = tmem_base + slot * kTsSlotCols;
            const uint64_t bd = umma_desc_sw128(b_st + j * kHalf * 128u);
#pragma unroll
            for (int ks = 0; ks < 8; ++ks)  // descriptor start address advances in 16-B units
              mma_bf16_ts_pair(d_tmem, a_tmem + 8u * ks,
                               bd + (uint64_t)(((ks >> 2) * half_tile + (ks & 3) * 32) >> 4),
                               idesc, ks != 0 ? 1u : 0u);
            mma_commit_pair_mc(bar_tfull(slot, grp), 0x3);
            if (STATS) st_issue += clock64() - w1;
            if (++slot == kTsSlots) slot = 0;
          }
          mma_commit_pair_mc(bar_empty(s), 0x3);  // both CTAs' stage s free again
          if (++s == S) { s = 0; ph ^= 1u; }
        }
        mma_commit_pair_mc(bar_afree, 0x1);
      }
      if (STATS && args.stats) {
        atomicAdd(args.stats + 0, (unsigned long long)st_acc);
        atomicAdd(args.stats + 1, (unsigned long long)st_full);
        atomicAdd(args.stats + 2, (unsigned long long)(clock64() - st_t0));
        atomicAdd(args.stats + 6, (unsigned long long)st_issue);
      }
    }
  } else if (warp < 8) {
    // ================= epilogue (both CTAs): group e drains the chunks of parity e =================
    const uint32_t qslot = warp & 3u;
    const uint32_t grp = warp >> 2;
    const uint32_t lanes = tmem_base + ((qslot * 32u) << 16);
    uint32_t t = 0, mine = 0, full_ph = 0;  // full_ph bit j: parity of (slot j, grp)'s next completion
    for (int32_t u = (int32_t)pair; u < n_units; u += (int32_t)n_pairs) {
      int32_t g, p;
      int64_t c0, c1;
      unit_decode(args, u, g, p, c0, c1);
      const int32_t q = g * 8 + (int32_t)rank * 4 + (int32_t)qslot;
      const int32_t lq = q < args.n_q ? __ldg(args.q_lens + q) : 0;
      WarpTopK<KR> topk;
      topk.init();
      const uint32_t tu = t;  // chunks (of both groups) before this unit
      const int64_t first = c0 + (int64_t)((grp - (t & 1u)) & 1u);
      t += (uint32_t)(c1 - c0);
      int32_t ld_next = (first < c1) ? __ldg(args.d_lens + first) : 0;
      for (int64_t c = first; c < c1; c += 2, ++mine) {
        const int32_t ld = ld_next;
        if (c + 2 < c1) ld_next = __ldg(args.d_lens + c + 2);
        // this chunk's 4 slots: uses 4 * (chunk counter) + j of the ring
        const uint32_t cidx = tu + (uint32_t)(c - c0);
        uint32_t slot = (kSub * cidx) % kTsSlots;
        float m4[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
#pragma unroll 1
        for (uint32_t j = 0; j < kSub; ++j) {
          long long e0 = STATS ? clock64() : 0;
          mbar_wait(bar_tfull(slot, grp), (full_ph >> slot) & 1u);
          full_ph ^= 1u << slot;
          long long e1 = STATS ? clock64() : 0;
          if (STATS) st_ewait += e1 - e0;
          tc_fence_after();
          // columns [0, SN/2): chunk rows (SN/2) j + n; [SN/2, SN): rows 128 + (SN/2) j + (n - SN/2)
          const int rem0 = ld - (int)(kHalf * j), rem1 = ld - 128 - (int)(kHalf * j);
#pragma unroll
          for (uint32_t h = 0; h < SN / 64; ++h) {
            uint32_t v[64];
            tmem_ld64_wait(lanes + slot * kTsSlotCols + 64u * h, v);
            if (rem1 >= (int)kHalf) {
              max64(v, m4);
            } else {
#pragma unroll
              for (int i = 0; i < 64; ++i) {
                const int n = (int)(64 * h) + i;
                const bool real = n < (int)kHalf ? n < rem0 : (n - (int)kHalf) < rem1;
                m4[i & 3] = fmaxf(m4[i & 3], real ? __uint_as_float(v[i]) : -INFINITY);
              }
            }
          }
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive_cluster(mapa_shared(bar_tempty(slot), 0));
          if (STATS) {
            st_drain += clock64() - e1;
            ++st_tiles;
          }
          if (++slot == kTsSlots) slot = 0;
        }
        const float m = fmaxf(fmaxf(m4[0], m4[1]), fmaxf(m4[2], m4[3]));
        float sv = ((int32_t)lane < lq) ? m : 0.0f;
#pragma unroll
        for (int o = 16; o >= 1; o >>= 1) sv += __shfl_xor_sync(0xffffffffu, sv, o);
        sv += 0.0f;  // canonical +0
        if constexpr (MODE == 0) {
          if (lane == 0 && q < args.n_q) args.scores[(int64_t)q * args.score_ld + c] = sv;
        } else {
          const uint64_t key = make_key(sv, args.id_base + c);
          if (key > topk.thresh) topk.insert(key, args.k, lane);
        }
      }
      if constexpr (MODE == 1) {
        uint64_t* dst = args.partial + (((int64_t)p * kEpiGroups + grp) * args.q_pad + q) * args.k;
#pragma unroll
        for (int r = 0; r < KR; ++r) {
          const int i = r * 32 + (int)lane;
          if (i < args.k) dst[i] = topk.v[r];
        }
      }
    }
  }

  if (STATS && warp < 8 && args.stats && lane == 0) {
    atomicAdd(args.stats + 3, (unsigned long long)st_drain);
    atomicAdd(args.stats + 4, (unsigned long long)st_ewait);
    atomicAdd(args.stats + 5, (unsigned long long)st_tiles);
  }
  tc_fence_before();
  cluster_sync();
  if (warp == kPairAllocWarp) {
    tc_fence_after();
    tmem_dealloc_pair(tmem_base, kTmemCols);
  }
}

}  // namespace hiper
