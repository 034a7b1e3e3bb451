// pooled_cs_sm100.cuh -- step a12 (BASELINE.json configs[4]) with the CHUNK tile stationary.
//
// The pooled limit case (Lq = Ld = 1: S(q, c) = <NORM(q), NORM(c)>, the cosine of pooled embeddings,
// PAPER.md:241, 385) is a dense GEMM S = Q C^T with K = dim and a fused per-query top-k.  The
// streaming kernel (pooled_sm100_pair.cuh) keeps neither operand resident at K = 768, so per K = 16
// step each CTA's shared memory is written with A and B (8 KB) and read for A (4 KB) and both tensor
// cores' B halves (8 KB): 160 B/clk against the 128 B/clk port -- a ~0.80 ceiling.
//
// Here a CTA pair keeps one 256-chunk tile resident (CTA r: its 128 chunk rows x dim, all K-blocks,
// 128B swizzle; 192 KB at dim 768) and streams every 256-query tile against it, so only the query
// operand moves: per K = 16 step 4 KB of A written + 4 KB of A read + 8 KB of B read = 128 B/clk,
// exactly the port.  The corpus is read from HBM once (each pair owns a contiguous range of chunk
// tiles: no L2 lockstep needed); the 4096 x 768 query block (6 MB) stays in L2.
//  * A stages are 32-dim K-blocks (8 KB per CTA, 64B swizzle) so 4 fit beside the resident chunk
//    tile: 3 stages of look-ahead (768 MMA cycles) cover the L2 latency.
//  * The next chunk tile streams into the resident region K-block by K-block as the last query tile
//    of the current one releases it (B_empty[kb] after its last MMA), i.e. the reload overlaps MMAs.
//  * The query changes every accumulator, so the per-query top-k lists cannot live in registers:
//    list (pair p, slot, query q) lives in global memory partial[p][slot][q_pad][k] and is owned by
//    one epilogue thread (the one holding q's TMEM lane in the group that drains q's tiles).  Per
//    tile the thread reads the list's k-th key and the shared bound gthr[q] (issued before it waits
//    for the accumulator), filters its 256 scores with one float compare per 64-column block, and
//    loads / updates / stores the list only on a hit (~0.07 per thread-tile at config 5).
//  * slot = 0 when the number of query tiles is even (tile t = ct * n_qt + qt goes to accumulator and
//    group t & 1 = qt & 1, so each query is always drained by the same group); otherwise slot = the
//    group (both groups see every query; separate lists, no races).  topk_merge.cuh merges the
//    P (or 2P) lists of each query.
#pragma once
#include "pooled_sm100_pair.cuh"

namespace hiper {

struct PooledCsArgs {
  int32_t n_q;        // real queries
  int32_t n_qtiles;   // ceil(n_q / 256)
  int32_t n_ctiles;   // ceil(n_chunks / tile_n)
  int32_t tile_n;     // chunks per tile = MMA N (multiple of 16, <= 256); CTA r holds tile_n / 2 rows
  int32_t n_parts;    // P = CTA pairs in the grid (pair p owns chunk tiles [p n_ct / P, (p+1) n_ct / P))
  int32_t num_kb;     // ceil(dim / 64): resident 64-dim K-blocks of the chunk tile
  int32_t k;          // top-k, k <= KP
  int32_t n_stages;   // A stages (a_cols-dim K-blocks, 128 x a_cols x 2 B per CTA)
  int32_t a_cols;     // 32 (64-B rows, SWIZZLE_64B) or 64 (128-B rows, SWIZZLE_128B)
  int32_t dbg;        // ablation (HIPER_POOLED_CS_DBG, results meaningless): bit 0 = no query TMA
                      // after the first S stages, bit 1 = no chunk TMA after the first tile,
                      // bit 2 = query stages placed below the resident chunk tile, bit 3 = the
                      // epilogue reads no TMEM, bit 4 = no list / bound loads before the wait, bit 5 = no
                      // query-tile rotation
  int32_t q_pad;      // n_qtiles * 256 (list row stride)
  int32_t two_slots;  // 1: lists per (pair, group, query) (odd n_qtiles); 0: per (pair, query)
  int64_t n_chunks;
  int64_t id_base;
  uint64_t* partial;           // [P][2][q_pad][k]
  unsigned long long* gthr;    // [q_pad] shared pruning bound (see PooledArgs::gthr), or nullptr
  unsigned long long* stats;   // HIPER_PIPE_STATS: [0] MMA wait acc, [1] wait A, [2] MMA total,
                               // [3] epilogue drain, [4] epilogue wait, [5] tiles, [6] wait B,
                               // [7] blocks past the threshold, [8] list loads
};

constexpr uint32_t kCsBBytes = 16384u;  // one resident 64-dim K-block at tile_n = 256: 128 rows x 128 B
constexpr uint32_t kCsABytes = 8192u;   // one A stage: 128 query rows x 32 dims x 2 B

// K-major operand in the canonical 64-byte-swizzled layout: rows of 32 bf16 (64 B), 8-row atoms of
// 512 B stacked along M (SBO = 512 B), LBO unused (1), version 1, layout type 4 (SWIZZLE_64B).
__device__ __forceinline__ uint64_t umma_desc_sw64(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)1 << 16;
  d |= (uint64_t)(512 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)4 << 61;
  return d;
}

template <int KP, int AC, bool STATS = false>
__global__ void __launch_bounds__(kMaxsimThreads, 1)
    pooled_cs_sm100_kernel(const __grid_constant__ CUtensorMap tmap_q32,
                           const __grid_constant__ CUtensorMap tmap_c, const PooledCsArgs args) {
  extern __shared__ uint8_t smem_raw[];
  using namespace ptx;
  const uint32_t warp = warp_id();
  const uint32_t lane = lane_id();
  const uint32_t rank = cluster_ctarank() & 1u;  // CTA within its pair (0 = leader)
  const uint32_t pair = cluster_id_x();
  const uint16_t pair_mask = 3u;

  const int NKB = args.num_kb, S = args.n_stages, NQT = args.n_qtiles, TN = args.tile_n;
  const uint32_t kbB = (uint32_t)TN * 64u;                 // one K-block of this CTA's TN / 2 rows
  const uint32_t base = (smem_u32(smem_raw) + 1023u) & ~1023u;
  constexpr int HPK = 64 / AC;                              // A stages per resident K-block
  const uint32_t aB = 256u * (uint32_t)AC;                 // one A stage: 128 rows x AC x 2 B
  const bool a_first = (args.dbg & 4) != 0;
  const uint32_t sB = a_first ? base + (uint32_t)S * aB : base;  // NKB x kbB, resident chunk tile
  const uint32_t sA = a_first ? base : sB + (uint32_t)NKB * kbB;  // S x aB query stages
  const uint32_t sBar = base + (uint32_t)NKB * kbB + (uint32_t)S * aB;
  auto bar_afull = [&](int s) { return sBar + 8u * s; };
  auto bar_aempty = [&](int s) { return sBar + 8u * (S + s); };
  auto bar_bfull = [&](int kb) { return sBar + 8u * (2 * S + kb); };
  auto bar_bempty = [&](int kb) { return sBar + 8u * (2 * S + NKB + kb); };
  auto bar_tfull = [&](int b) { return sBar + 8u * (2 * S + 2 * NKB + b); };
  auto bar_tempty = [&](int b) { return sBar + 8u * (2 * S + 2 * NKB + 2 + b); };
  const uint32_t sTmemPtr = sBar + 8u * (2 * S + 2 * NKB + 4);
  uint32_t* tmem_ptr_generic = reinterpret_cast<uint32_t*>(smem_raw + (sTmemPtr - smem_u32(smem_raw)));

  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(bar_afull(s), 1);
      mbar_init(bar_aempty(s), 1);
    }
    for (int kb = 0; kb < NKB; ++kb) {
      mbar_init(bar_bfull(kb), 1);
      mbar_init(bar_bempty(kb), 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(bar_tfull(b), 1);
      mbar_init(bar_tempty(b), 8);
    }
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

  // pair p visits the query tiles in the order p, p + 1, ... (mod n_qtiles): the pairs run in step,
  // and without the rotation all of them would fetch the same query K-block from the same L2 lines
  const int32_t qrot = (args.dbg & 32) ? 0 : (int32_t)(pair % (uint32_t)NQT);
  auto qtile = [&](int32_t qt) { return qt + qrot < NQT ? qt + qrot : qt + qrot - NQT; };
  const int32_t t0 = (int32_t)((int64_t)pair * args.n_ctiles / args.n_parts);
  const int32_t t1 = (int32_t)((int64_t)(pair + 1) * args.n_ctiles / args.n_parts);

  if (warp == kPairProducerWarp) {
    if (lane == 0) {
      prefetch_tmap(&tmap_q32);
      prefetch_tmap(&tmap_c);
      int s = 0;
      uint32_t ph = 0, bph = 0;
      for (int32_t ct = t0; ct < t1; ++ct, bph ^= 1u) {
        for (int32_t qt = 0; qt < NQT; ++qt) {
          const int32_t qrow0 = qtile(qt) * 256 + (int32_t)rank * 128;
          for (int kb = 0; kb < NKB; ++kb) {
            if (qt == 0) {  // the chunk tile's K-block, once the previous tile's last MMA read it
              mbar_wait(bar_bempty(kb), bph ^ 1u);
              if ((args.dbg & 2) && ct > t0) {
                if (rank == 0) mbar_arrive(bar_bfull(kb));
              } else {
                if (rank == 0) mbar_arrive_expect_tx(bar_bfull(kb), 2u * kbB);
                tma_load_2d_pair(sB + (uint32_t)kb * kbB, &tmap_c, mapa_shared(bar_bfull(kb), 0),
                                 kb * 64, ct * TN + (int32_t)rank * (TN / 2));
              }
            }
#pragma unroll
            for (int hh = 0; hh < HPK; ++hh) {
              mbar_wait(bar_aempty(s), ph ^ 1u);
              if ((args.dbg & 1) && (ct > t0 || qt > 0 || kb * HPK + hh >= S)) {
                if (rank == 0) mbar_arrive(bar_afull(s));
              } else {
                if (rank == 0) mbar_arrive_expect_tx(bar_afull(s), 2u * aB);
                tma_load_2d_pair(sA + (uint32_t)s * aB, &tmap_q32, mapa_shared(bar_afull(s), 0),
                                 (kb * HPK + hh) * AC, qrow0);
              }
              if (++s == S) { s = 0; ph ^= 1u; }
            }
          }
        }
      }
    }
  } else if (warp == kPairMmaWarp) {
    if (rank == 0 && lane == 0) {
      // a lean issue loop: the single MMA thread's per-stage overhead has to stay well below the
      // stage's MMA time (a runtime divide here cost 35% of the tensor rate at AC = 32)
      const uint32_t idesc = idesc_bf16_f32(256, (uint32_t)TN);
      const uint64_t a_hi = (AC == 32 ? umma_desc_sw64(0) : umma_desc_sw128(0));
      const uint64_t b_hi = umma_desc_sw128(0);
      int s = 0;
      uint32_t ph = 0, bph = 0, t = 0;
      long long st_acc = 0, st_a = 0, st_b = 0, w0 = 0;
      const long long st_t0 = STATS ? clock64() : 0;
      for (int32_t ct = t0; ct < t1; ++ct, bph ^= 1u) {
        for (int32_t qt = 0; qt < NQT; ++qt, ++t) {
          const uint32_t acc = t & 1u, tph = (t >> 1) & 1u;
          if (STATS) w0 = clock64();
          mbar_wait(bar_tempty(acc), tph ^ 1u);
          if (STATS) st_acc += clock64() - w0;
          tc_fence_after();
          const uint32_t d_tmem = tmem_base + acc * kAccStride;
          const bool last_q = qt == NQT - 1;
          for (int kb = 0; kb < NKB; ++kb) {
            if (qt == 0) {
              if (STATS) w0 = clock64();
              mbar_wait(bar_bfull(kb), bph);
              if (STATS) st_b += clock64() - w0;
            }
            const uint32_t b_lo = (sB + (uint32_t)kb * kbB) >> 4;
#pragma unroll
            for (int hh = 0; hh < HPK; ++hh) {
              if (STATS) w0 = clock64();
              mbar_wait(bar_afull(s), ph);
              if (STATS) st_a += clock64() - w0;
              tc_fence_after();
              const uint32_t a_lo = (sA + (uint32_t)s * aB) >> 4;
#pragma unroll
              for (int kk = 0; kk < AC / 16; ++kk)
                mma_bf16_ss_pair(d_tmem, a_hi | (uint64_t)(a_lo + 2u * kk),
                                 b_hi | (uint64_t)(b_lo + 4u * hh + 2u * kk), idesc,
                                 (kb | hh | kk) != 0 ? 1u : 0u);
              mma_commit_pair_mc(bar_aempty(s), pair_mask);
              if (++s == S) { s = 0; ph ^= 1u; }
            }
            if (last_q) mma_commit_pair_mc(bar_bempty(kb), pair_mask);
          }
          mma_commit_pair_mc(bar_tfull(acc), pair_mask);
        }
      }
      if (STATS && args.stats) {
        atomicAdd(args.stats + 0, (unsigned long long)st_acc);
        atomicAdd(args.stats + 1, (unsigned long long)st_a);
        atomicAdd(args.stats + 2, (unsigned long long)(clock64() - st_t0));
        atomicAdd(args.stats + 6, (unsigned long long)st_b);
      }
    }
  } else if (warp < 8) {
    const uint32_t qslot = warp & 3u;
    const uint32_t grp = warp >> 2;
    const uint32_t taddr_base = tmem_base + ((qslot * 32u) << 16) + grp * kAccStride;
    const uint32_t tempty_leader = mapa_shared(bar_tempty(grp), 0);
    const int32_t k = args.k;
    const uint32_t slot = args.two_slots ? grp : 0u;
    const int32_t qrow = (int32_t)rank * 128 + (int32_t)(qslot * 32u + lane);
    uint64_t* lists = args.partial + ((int64_t)pair * kEpiGroups + slot) * args.q_pad * k;
    // this thread owns the lists of its TMEM lane's query in every query tile it drains: empty them
    for (int32_t qt = (args.two_slots ? 0 : (int32_t)grp); qt < NQT; qt += (args.two_slots ? 1 : 2)) {
      const int32_t q = qtile(qt) * 256 + qrow;
      if (q < args.n_q)
        for (int m = 0; m < k; ++m) lists[(int64_t)q * k + m] = 0ull;
    }
    long long st_drain = 0, st_ewait = 0, st_tiles = 0, st_any = 0, st_loads = 0;
    uint32_t t = 0, mine = 0;
    for (int32_t ct = t0; ct < t1; ++ct) {
      const int64_t cbase = (int64_t)ct * TN;
      const int64_t left = args.n_chunks - cbase;
      const int32_t ncols = (args.dbg & 8) ? 0 : (left < TN ? (int32_t)left : TN);
      for (int32_t qt = 0; qt < NQT; ++qt, ++t) {
        if ((t & 1u) != grp) continue;
        const int32_t q = qtile(qt) * 256 + qrow;
        const bool valid = q < args.n_q;
        uint64_t* L = lists + (int64_t)(valid ? q : 0) * k;
        // the list's k-th key and the shared bound, loaded before the accumulator wait
        uint64_t thr = valid ? ((args.dbg & 16) ? 0ull : L[k - 1]) : ~0ull;
        uint64_t gth = (valid && args.gthr != nullptr && !(args.dbg & 16))
                           ? *reinterpret_cast<volatile unsigned long long*>(args.gthr + q) : 0ull;
        uint64_t lim = thr > gth ? thr : gth;
        float thr_f = valid ? pooled_thr_score(lim) : INFINITY;
        long long e0 = STATS ? clock64() : 0;
        mbar_wait(bar_tfull(grp), mine & 1u);
        long long e1 = STATS ? clock64() : 0;
        if (STATS) st_ewait += e1 - e0;
        tc_fence_after();
        uint64_t v[KP];
        bool loaded = false;
        for (int32_t col = 0; col < ncols; col += 64) {
          uint32_t r[64];
          tmem_ld64_wait(taddr_base + (uint32_t)col, r);
          const int32_t nj = ncols - col;
          bool any;
          if (nj >= 64) {
            float m4[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
            max64(r, m4);
            any = fmaxf(fmaxf(m4[0], m4[1]), fmaxf(m4[2], m4[3])) >= thr_f;
          } else {
            any = true;
          }
          uint64_t hits = 0ull;
          if (any) {
            if (STATS) ++st_any;
#pragma unroll
            for (int j = 0; j < 64; ++j)
              hits |= (uint64_t)(__uint_as_float(r[j]) >= thr_f && j < nj) << j;
          }
          if (hits) {  // rare: fetch the list once per tile, insert the keys above max(k-th, bound)
            float xs[64];
#pragma unroll
            for (int j = 0; j < 64; ++j) xs[j] = __uint_as_float(r[j]) + 0.0f;
            if (!loaded) {
              if (STATS) ++st_loads;
#pragma unroll
              for (int m = 0; m < KP; ++m) v[m] = m < k ? L[m] : 0ull;
              loaded = true;
            }
            while (hits) {
              const int j = __ffsll((long long)hits) - 1;
              hits &= hits - 1;
              uint64_t key = make_key(xs[j], args.id_base + cbase + col + j);
              if (key > lim) {
#pragma unroll
                for (int m = 0; m < KP; ++m) {
                  const uint64_t hi = v[m] > key ? v[m] : key;
                  key = v[m] > key ? key : v[m];
                  v[m] = hi;
                }
                uint64_t nt = 0ull;
#pragma unroll
                for (int m = 0; m < KP; ++m)
                  if (m == k - 1) nt = v[m];
                thr = nt;
                lim = thr > gth ? thr : gth;
                thr_f = pooled_thr_score(lim);
              }
            }
          }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive_cluster(tempty_leader);
        if (STATS) {
          st_drain += clock64() - e1;
          ++st_tiles;
        }
        if (loaded) {  // write the list back; publish its k-th key as the query's shared bound
#pragma unroll
          for (int m = 0; m < KP; ++m)
            if (m < k) L[m] = v[m];
          if (args.gthr != nullptr && thr > gth) atomicMax(args.gthr + q, (unsigned long long)thr);
        }
        ++mine;
      }
    }
    if (STATS && args.stats) {
      if (lane == 0) {
        atomicAdd(args.stats + 3, (unsigned long long)st_drain);
        atomicAdd(args.stats + 4, (unsigned long long)st_ewait);
        atomicAdd(args.stats + 5, (unsigned long long)st_tiles);
      }
      atomicAdd(args.stats + 7, (unsigned long long)st_any);
      atomicAdd(args.stats + 8, (unsigned long long)st_loads);
    }
  }

  tc_fence_before();
  cluster_sync();
  if (warp == kPairAllocWarp) {
    tc_fence_after();
    tmem_dealloc_pair(tmem_base, kTmemCols);
  }
}

}  // namespace hiper
