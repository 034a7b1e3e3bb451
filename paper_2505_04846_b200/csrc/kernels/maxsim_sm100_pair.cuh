// maxsim_sm100_pair.cuh -- steps a3-a6 on a CTA pair (cta_group::2): the production MaxSim kernel.
//
//   S(q, c) = sum_{i < len_q} max_{j < len_c} < q_i , d_{c,j} >       (§2.2, Fig.3B
//                                                                    PAPER.md:228)
//
// Same method and epilogue as maxsim_sm100.cuh, but two SMs of a TPC cooperate on every MMA:
//  * a cluster of 2 CTAs owns a "row-group pair" of 8 queries (256 query-token rows): CTA r keeps
//    the A tile of queries 8g+4r .. 8g+4r+3 (128 rows) resident in its shared memory;
//  * per chunk, CTA r TMA-loads only token rows [r*ld_pad/2, (r+1)*ld_pad/2) of the chunk, so each SM
//    fills half as many B bytes per MMA FLOP as the single-CTA kernel (L2->SMEM and SMEM-port
//    traffic halved: the profiled limiter of the M = 128 kernel);
//  * the leader CTA's single MMA thread issues tcgen05.mma.cta_group::2 with M = 256, N = ld_pad,
//    K = 16: the hardware reads A and B halves from both CTAs' shared memory and writes each CTA's
//    128 accumulator rows into that CTA's TMEM (128 lanes x ld_pad fp32 columns);
//  * each CTA's two epilogue warpgroups drain their own TMEM exactly as in the single-CTA kernel and
//    release the accumulator to the leader with a cluster-scope mbarrier arrive.
// Barriers: full[s] / a_full[b] / t_empty[b] live in the leader (both CTAs' TMA complete_tx and both
// CTAs' epilogue arrivals land there); empty[s] / a_empty[b] / t_full[b] exist in both CTAs and are
// signalled by the leader's multicast tcgen05.commit.
#pragma once
#include "maxsim_sm100.cuh"

namespace hiper {

// DBG (ablation builds only, selected by HIPER_DEBUG_MODE): 0 = production; 1 = epilogue skips the
// TMEM reads and reductions (measures the TMA + MMA pipeline alone); 2 = additionally no chunk TMA
// after the first stage fill (measures MMA issue alone); 3 = no chunk TMA after the first stage fill
// but the full epilogue (measures MMA + epilogue without the L2 feed); 4 = mode 2 with every
// chunk's K loop issued twice into its accumulator (per-chunk fixed costs vs MMA time).  DBG != 0
// results are meaningless.
// warps 0-7: epilogue groups 0/1; 8: TMEM allocator; 9: spare; 10: TMA producer; 11: MMA issuer
constexpr uint32_t kPairAllocWarp = 8, kPairProducerWarp = 10, kPairMmaWarp = 11;

// L2 lockstep.  All pairs of a wave stream the same corpus partition(s); left alone they drift
// apart by more than the L2 can hold (measured: 5.6 TB of DRAM reads per launch for a 65.5 GB
// corpus at Q = 1024).  Each leader publishes its position -- the number of chunks it has streamed
// so far, continuous across its units (units are equal to within one chunk) -- every 16 chunks and
// waits while it is more than `window` chunks ahead of the slowest pair, so the chunks in flight
// across the GPU stay inside a few MB of L2.  (An earlier (unit << 20 | offset) position turned every
// unit boundary into a grid-wide barrier.)  Finished pairs publish ~0u.
__device__ __forceinline__ void lockstep_publish(uint32_t* progress, uint32_t pair, uint32_t pos) {
  *reinterpret_cast<volatile uint32_t*>(progress + pair) = pos;
}
__device__ __forceinline__ void lockstep_wait(const uint32_t* progress, uint32_t n_pairs, uint32_t pos,
                                              uint32_t window) {
  const long long t0 = clock64();
  while (true) {
    // 16 independent loads in flight per round (a plain loop waits out each load's L2 latency in
    // turn: ~n_pairs round trips per check)
    uint32_t mn = 0xFFFFFFFFu;
    for (uint32_t j0 = 0; j0 < n_pairs; j0 += 16) {
      uint32_t v[16];
#pragma unroll
      for (int q = 0; q < 16; ++q)
        v[q] = j0 + q < n_pairs ? *reinterpret_cast<const volatile uint32_t*>(progress + j0 + q) : 0xFFFFFFFFu;
#pragma unroll
      for (int q = 0; q < 16; ++q) mn = min(mn, v[q]);
    }
    if ((uint64_t)pos <= (uint64_t)mn + window) return;
    __nanosleep(200);
    if (clock64() - t0 > HIPER_WATCHDOG_CYCLES) ptx::hiper_watchdog_fail("lockstep", pos, mn);
  }
}

// The same wait by a whole warp: lane l scans the words l, l + 32, ... and the minimum is a butterfly,
// so one check costs ~one L2 round trip instead of n_pairs dependent-issue loads by one thread.
__device__ __forceinline__ void lockstep_wait_warp(const uint32_t* progress, uint32_t n_pairs, uint32_t pos,
                                                   uint32_t window, uint32_t lane) {
  const long long t0 = clock64();
  while (true) {
    uint32_t mn = 0xFFFFFFFFu;
    for (uint32_t j = lane; j < n_pairs; j += 32)
      mn = min(mn, *reinterpret_cast<const volatile uint32_t*>(progress + j));
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) mn = min(mn, __shfl_xor_sync(0xffffffffu, mn, o));
    if ((uint64_t)pos <= (uint64_t)mn + window) return;
    __nanosleep(200);
    if (clock64() - t0 > HIPER_WATCHDOG_CYCLES) ptx::hiper_watchdog_fail("lockstep", pos, mn);
  }
}

// PACKED (N4): the slots are the tiles of a length-bucketed packed corpus (MaxsimArgs::recs): the MMA
// N is the tile's n_rows, and the epilogue reduces each chunk over its own column segment.
// STATS: HIPER_PIPE_STATS instrumentation compiled in (diagnostics builds only; the production
// instantiation carries none of it -- the kernel's hot loops are instruction-cache sensitive).
// QW: warps (32 token rows each) per query: 1 (q_max_len <= 32), 2 (<= 64), 4 (<= 128).
// H: MMA halves per chunk: 1 (ld_pad <= 256), 2 (256 < ld_pad <= 512; half h = rows [256h, ...)).
template <int MODE, int KR, int DBG = 0, bool PACKED = false, bool STATS = false, int QW = 1, int H = 1>
__global__ void __launch_bounds__(kMaxsimThreads, 1)
    maxsim_sm100_pair_kernel(const __grid_constant__ CUtensorMap tmap_q,
                             const __grid_constant__ CUtensorMap tmap_d, const MaxsimArgs args) {
  static_assert(QW == 1 || QW == 2 || QW == 4, "QW");
  static_assert(H == 1 || (H == 2 && !PACKED), "two-half chunks are dense-layout only");
  static_assert(MODE != 2 || (QW == 1 && H == 1), "argmax capture: q_max_len <= 32, ld_pad <= 256");
  extern __shared__ uint8_t smem_raw[];
  using namespace ptx;
  const uint32_t warp = warp_id();
  const uint32_t lane = lane_id();
  const uint32_t rank = cluster_ctarank();  // 0 = leader
  const uint32_t pair = cluster_id_x();
  const uint32_t n_pairs = nclusters_x();

  const uint32_t base = (smem_u32(smem_raw) + 1023u) & ~1023u;
  const uint32_t sA = base;                            // a_bufs x a_bytes (this CTA's 128 query rows)
  const uint32_t sB = sA + args.a_bufs * args.a_bytes;  // n_stages x stage_bytes
  const uint32_t sBar = sB + args.n_stages * args.stage_bytes;
  const int S = args.n_stages;
  auto bar_full = [&](int s) { return sBar + 8u * s; };
  auto bar_empty = [&](int s) { return sBar + 8u * (S + s); };
  auto bar_afull = [&](int b) { return sBar + 8u * (2 * S + b); };
  auto bar_aempty = [&](int b) { return sBar + 8u * (2 * S + 2 + b); };
  auto bar_tempty = [&](int b) { return sBar + 8u * (2 * S + 4 + b); };
  auto bar_tfull = [&](int b) { return sBar + 8u * (2 * S + 6 + b); };  // [acc + 2 * group] (H = 2)
  const uint32_t sTmemPtr = sBar + 8u * (2 * S + 10);
  const uint32_t sMeta = sTmemPtr + 16u;  // [S] u32: MMA N per stage (packed corpus)
  const uint32_t sRing = sBar + 512u;     // [2][32] x {w0, row0}: producer's tile batches (packed)
  // [2 groups][2 buffers][4 warps][16] fp32: per-warp partial sums of a query that spans QW warps
  float* xsum = reinterpret_cast<float*>(smem_raw + (sBar + 1024u - smem_u32(smem_raw)));
  uint32_t* tmem_ptr_generic =
      reinterpret_cast<uint32_t*>(smem_raw + (sTmemPtr - smem_u32(smem_raw)));

  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(bar_full(s), 1);   // leader's producer arrive (+ both CTAs' tx bytes)
      mbar_init(bar_empty(s), 1);  // leader's multicast commit
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(bar_afull(b), 1);
      mbar_init(bar_aempty(b), 1);
      mbar_init(bar_tempty(b), 8);  // 4 warps of the draining epilogue group in each of the 2 CTAs
    }
    for (int b = 0; b < 4; ++b) mbar_init(bar_tfull(b), 1);
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
  // PDL: the set-up above overlapped the previous kernel's tail; its outputs (the query / doc
  // layouts, lengths) are read only after this point.
  grid_dependency_wait();

  const int32_t n_units = args.n_groups * args.n_parts;
  long long st_drain_g = 0, st_ewait_g = 0, st_tiles_g = 0;  // HIPER_PIPE_STATS (epilogue warps)
  const uint32_t kb_bytes = args.box_rows * 128u;  // one 64-dim K-block of this CTA's rows
  // MMA N and this CTA's first row of half h of a dense chunk
  auto half_n = [&](int h) -> uint32_t {
    return H == 1 ? (uint32_t)args.ld_pad : (h == 0 ? 256u : (uint32_t)args.ld_pad - 256u);
  };
  auto a_slot = [&](uint32_t it, uint32_t& ab, uint32_t& aph) {
    ab = args.a_bufs == 2 ? (it & 1u) : 0u;
    aph = args.a_bufs == 2 ? ((it >> 1) & 1u) : (it & 1u);
  };

  if (warp == kPairProducerWarp) {
    // ================= TMA producer (both CTAs) =================
    // The whole warp walks the units; lane 0 waits on barriers and issues the TMA.  For a packed
    // corpus the warp loads the tile descriptors 32 at a time, one batch ahead, so no dependent
    // global load sits between two stages (a miss costs ~1 us, about two tiles of MMA work).
    if (lane == 0) {
      prefetch_tmap(&tmap_q);
      prefetch_tmap(&tmap_d);
    }
    int s = 0;
    uint32_t ph = 0, it = 0, streamed = 0;  // streamed: chunks of this pair's finished units
    for (int32_t u = (int32_t)pair; u < n_units; u += (int32_t)n_pairs, ++it) {
      int32_t g, p;
      int64_t c0, c1;
      unit_decode(args, u, g, p, c0, c1);
      if (lane == 0) {
        uint32_t ab, aph;
        a_slot(it, ab, aph);
        mbar_wait(bar_aempty(ab), aph ^ 1u);
        if (rank == 0) mbar_arrive_expect_tx(bar_afull(ab), 2u * args.a_bytes);
        const uint32_t afull_leader = mapa_shared(bar_afull(ab), 0);
        for (int kb = 0; kb < args.num_kb; ++kb)
          tma_load_2d_pair(sA + ab * args.a_bytes + kb * 16384u, &tmap_q, afull_leader, kb * 64,
                           (int32_t)((2 * g + (int32_t)rank) * 128));
      }
      // packed: (w0, row0) of 32 tiles at a time land in an SMEM ring by cp.async, one batch ahead
      auto load_batch = [&](int64_t cb, uint32_t slot) {
        const int64_t ci = cb + lane;
        if (ci < c1) {
          const uint32_t dst = sRing + slot * 256u + lane * 8u;
          cp_async4(dst, args.recs + ci * 32);
          cp_async4(dst + 4u, args.recs + ci * 32 + 4);
        }
        cp_async_commit();
      };
      if constexpr (PACKED) load_batch(c0, 0u);
      for (int64_t c = c0; c < c1; ++c) {
        int32_t brow;
        uint32_t nrows = (uint32_t)args.ld_pad;
        if constexpr (PACKED) {
          const uint32_t j = (uint32_t)((c - c0) & 31), b = (uint32_t)((c - c0) >> 5);
          if (j == 0) {
            load_batch(c + 32, (b + 1) & 1u);
            cp_async_wait<1>();  // batch b (issued 32 tiles ago) has landed
            __syncwarp();
          }
          const uint32_t e = sRing + (b & 1u) * 256u + j * 8u;
          nrows = ld_shared_u32(e) & 0xFFFFu;
          brow = (int32_t)ld_shared_u32(e + 4u) + (int32_t)rank * (int32_t)(nrows >> 1);
        } else {
          brow = (int32_t)(c * args.ld_pad + (int64_t)rank * (half_n(0) >> 1));
        }
        if (args.progress != nullptr && rank == 0 && ((c - c0) & args.ls_mask) == 0) {  // warp-uniform
          const uint32_t pos = streamed + (uint32_t)(c - c0);
          if (lane == 0) lockstep_publish(args.progress, pair, pos);
          lockstep_wait_warp(args.progress, n_pairs, pos, (uint32_t)args.window, lane);
        }
        if (lane == 0) {
#pragma unroll
          for (int h = 0; h < H; ++h) {
            // one stage = this CTA's rows of one whole chunk (half), all K-blocks
            mbar_wait(bar_empty(s), ph ^ 1u);
            if constexpr (PACKED) st_shared_u32(sMeta + 4u * s, nrows);  // MMA N of this stage
            if ((DBG == 2 || DBG == 3 || DBG == 4) && (c > c0 || it > 0)) {
              if (rank == 0) mbar_arrive(bar_full(s));
            } else {
              if (rank == 0) mbar_arrive_expect_tx(bar_full(s), 2u * args.stage_bytes);
              const uint32_t full_leader = mapa_shared(bar_full(s), 0);
              // half 1 starts at row 256 of the chunk; this CTA takes the second half of its N rows
              const int32_t row = H == 1 ? brow
                                         : (int32_t)(c * args.ld_pad + h * 256 + (int64_t)rank * (half_n(h) >> 1));
              for (int kb = 0; kb < args.num_kb; ++kb)
                tma_load_2d_pair(sB + s * args.stage_bytes + kb * kb_bytes, &tmap_d, full_leader,
                                 kb * 64, row);
            }
            if (++s == S) { s = 0; ph ^= 1u; }
          }
        }
        __syncwarp();
      }
      streamed += (uint32_t)(c1 - c0);
    }
    if (lane == 0 && args.progress != nullptr && rank == 0) lockstep_publish(args.progress, pair, 0xFFFFFFFFu);
  } else if (warp == kPairMmaWarp) {
    // ================= MMA issuer: leader CTA, single thread =================
    // (highest warp id: the SMSP arbiter favours it over the epilogue warps sharing its SMSP)
    if (rank == 0 && lane == 0) {
      const uint32_t idesc = idesc_bf16_f32(256, half_n(0));
      int s = 0;
      uint32_t ph = 0, it = 0, t = 0;  // t: accumulator turns (chunk halves) so far
      long long st_acc = 0, st_full = 0;
      const long long st_t0 = clock64();
      for (int32_t u = (int32_t)pair; u < n_units; u += (int32_t)n_pairs, ++it) {
        int32_t g, p;
        int64_t c0, c1;
        unit_decode(args, u, g, p, c0, c1);
        uint32_t ab, aph;
        a_slot(it, ab, aph);
        mbar_wait(bar_afull(ab), aph);
        tc_fence_after();
        const uint32_t a_tile = sA + ab * args.a_bytes;
        for (int64_t c = c0; c < c1; ++c) {
#pragma unroll
          for (int h = 0; h < H; ++h, ++t) {
            const uint32_t acc = t & 1u, tph = (t >> 1) & 1u;
            long long w0 = (STATS && args.stats) ? clock64() : 0;
            mbar_wait(bar_tempty(acc), tph ^ 1u);
            if (STATS && args.stats) {
              st_acc += clock64() - w0;
              w0 = clock64();
            }
            tc_fence_after();
            const uint32_t d_tmem = tmem_base + acc * kAccStride;
            mbar_wait(bar_full(s), ph);
            if (STATS && args.stats) st_full += clock64() - w0;
            tc_fence_after();
            uint32_t idesc_c = idesc;
            if constexpr (PACKED)  // MMA N = this tile's packed rows (written by the producer)
              idesc_c = idesc_bf16_f32(256, ld_shared_u32(sMeta + 4u * s));
            if constexpr (H == 2) idesc_c = idesc_bf16_f32(256, half_n(h));
            const uint32_t b_st = sB + s * args.stage_bytes;
            for (int rep = 0; rep < (DBG == 4 ? 2 : 1); ++rep)  // DBG 4: each chunk's K loop twice
            for (int kb = 0; kb < args.num_kb; ++kb) {
              const uint32_t a_kb = a_tile + kb * 16384u;
              const uint32_t b_kb = b_st + kb * kb_bytes;
#pragma unroll
              for (int kk = 0; kk < 4; ++kk)
                mma_bf16_ss_pair(d_tmem, umma_desc_sw128(a_kb + kk * 32),
                                 umma_desc_sw128(b_kb + kk * 32), idesc_c, (rep | kb | kk) != 0 ? 1u : 0u);
            }
            mma_commit_pair_mc(bar_empty(s), 0x3);  // both CTAs' stage s free again
            if (++s == S) { s = 0; ph ^= 1u; }
            // both CTAs' accumulator rows ready; H = 2: the barrier of (half, draining group)
            mma_commit_pair_mc(bar_tfull(H == 1 ? acc : acc + 2u * ((t >> 1) & 1u)), 0x3);
          }
        }
        mma_commit_pair_mc(bar_aempty(ab), 0x3);
      }
      if (STATS && args.stats) {
        atomicAdd(args.stats + 0, (unsigned long long)st_acc);
        atomicAdd(args.stats + 1, (unsigned long long)st_full);
        atomicAdd(args.stats + 2, (unsigned long long)(clock64() - st_t0));
      }
    }
  } else if (warp < 8) {
    // ================= epilogue (both CTAs, each on its own 128 TMEM lanes) =================
    // warp w reads TMEM lanes 32*(w%4)..+31 (the hardware's lane-quarter rule).  Group e drains the
    // chunks of parity e; with H = 2 it drains both halves of its chunk (accumulators 0 and 1).
    const uint32_t qslot = warp & 3u;
    const uint32_t grp = warp >> 2;
    const uint32_t qc = qslot / QW, part = qslot % QW;  // query within this CTA, its 32-row part
    const uint32_t lanes = tmem_base + ((qslot * 32u) << 16);
    const uint32_t taddr_base = lanes + grp * kAccStride;
    const uint32_t tempty_leader = mapa_shared(bar_tempty(grp), 0);
    uint32_t t = 0, mine = 0;
    // a query spanning QW warps: its warps' sums meet in shared memory (double-buffered by chunk)
    auto combine = [&](float v, bool write, uint32_t idx) -> float {
      if constexpr (QW == 1) {
        return v;
      } else {
        float* xs = xsum + (grp * 2u + (mine & 1u)) * 64u;
        if (write) xs[qslot * 16u + idx] = v;
        named_bar_sync(1u + grp * 4u + qc, 32u * QW);
        if (part == 0 && write) {
          float tsum = xs[qc * QW * 16u + idx];
#pragma unroll
          for (int w = 1; w < QW; ++w) tsum += xs[(qc * QW + w) * 16u + idx];
          v = tsum;
        }
        return v;
      }
    };
    for (int32_t u = (int32_t)pair; u < n_units; u += (int32_t)n_pairs) {
      int32_t g, p;
      int64_t c0, c1;
      unit_decode(args, u, g, p, c0, c1);
      const int32_t q = g * (8 / QW) + (int32_t)rank * (4 / QW) + (int32_t)qc;
      const int32_t lq = q < args.n_q ? __ldg(args.q_lens + q) : 0;
      const bool tok_real = (int32_t)(part * 32u + lane) < lq;
      WarpTopK<KR> topk;
      topk.init();
      const int64_t first = c0 + (int64_t)((grp - (t & 1u)) & 1u);
      t += (uint32_t)(c1 - c0);
      if constexpr (PACKED) {
        // Tile columns = 16 groups of 16, each inside one chunk.  Pass 1 reads the tile with the
        // same x64 TMEM loads as the dense kernel and keeps one max per group; pass 2 turns
        // them into per-chunk maxima (suffix max inside each chunk); pass 3 finishes each chunk.
        // The tile's 128-B record is one coalesced warp load (lane i <- word i), issued two of this
        // group's tiles (four MMA periods) ahead, so its DRAM latency never reaches the drain.
        auto load_rec = [&](int64_t ci) { return ci < c1 ? __ldg(args.recs + ci * 32 + lane) : 0u; };
        uint32_t rec_n1 = load_rec(first), rec_n2 = load_rec(first + 2);
        for (int64_t c = first; c < c1; c += 2, ++mine) {
          const uint32_t rec = rec_n1;
          rec_n1 = rec_n2;
          rec_n2 = load_rec(c + 4);
          const uint32_t w0 = __shfl_sync(0xffffffffu, rec, 0);
          const uint32_t gstart = __shfl_sync(0xffffffffu, rec, 1);
          const int32_t n_grp = (int32_t)(w0 & 0xFFFFu) >> 4;  // column groups in use
          long long e0 = (STATS && args.stats) ? clock64() : 0;
          mbar_wait(bar_tfull(grp), mine & 1u);
          long long e1 = (STATS && args.stats) ? clock64() : 0;
          if (STATS && args.stats) st_ewait_g += e1 - e0;
          tc_fence_after();
          // Pass 1: one running max per column group of 16 -- 4 independent FMNMX3 chains per
          // 64-column TMEM load, the dense kernel's instruction mix.  No column is masked: the
          // padding rows of a chunk's last 16-row group repeat its last real row (the packed layout
          // build, pack_pad_replicate_kernel), and a repeated column cannot change a maximum, so the
          // group max is the max over the chunk's real columns (reading R2) with no tail re-reads.
          float m16[16];
          bool released = false;  // early release after the last TMEM load (see the dense path)
#pragma unroll
          for (int blk = 0; blk < 4; ++blk) {
            if (blk * 4 < n_grp) {
              uint32_t v[64];
              tmem_ld64_wait(taddr_base + (uint32_t)(blk * 64), v);
              if (blk == ((n_grp - 1) >> 2) && !args.late_release) {
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive_cluster(tempty_leader);
                released = true;
              }
#pragma unroll
              for (int gg = 0; gg < 4; ++gg) {
                float a0 = fmaxf(__uint_as_float(v[gg * 16]), __uint_as_float(v[gg * 16 + 1]));
#pragma unroll
                for (int i = 2; i < 16; i += 2)
                  a0 = fmaxf(fmaxf(a0, __uint_as_float(v[gg * 16 + i])), __uint_as_float(v[gg * 16 + i + 1]));
                m16[blk * 4 + gg] = a0;
              }
            } else {
#pragma unroll
              for (int gg = 0; gg < 4; ++gg) m16[blk * 4 + gg] = -INFINITY;
            }
          }
          if (!released) {
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive_cluster(tempty_leader);  // TMEM drained: release the accumulator
          }
          if (STATS && args.stats) {
            st_drain_g += clock64() - e1;
            ++st_tiles_g;
          }
          // Pass 2: suffix max inside each chunk -> m16[first group of a chunk] = the chunk maximum
          // (start bits are set for every group >= n_grp, so unused groups never merge into a chunk)
#pragma unroll
          for (int gi = 14; gi >= 0; --gi)
            m16[gi] = ((gstart >> (gi + 1)) & 1u) ? m16[gi] : fmaxf(m16[gi], m16[gi + 1]);
          // Pass 3: the masked sum over query tokens of all 16 groups at once, by a transposed
          // butterfly (a reduce-scatter by shuffles): each round halves the groups a lane carries, and
          // lane l ends with the sum of group l >> 1.  Every group's sum is built from exactly the
          // dense kernel's butterfly pairings (xor 16, 8, 4, 2, 1; fp add is commutative), so the
          // scores are bitwise those of the dense layout -- in straight-line code instead of 16
          // branch-guarded butterflies (the kernel's hot loops are instruction-cache sensitive).
          float x[16];
#pragma unroll
          for (int gi = 0; gi < 16; ++gi) x[gi] = tok_real ? m16[gi] : 0.0f;
#pragma unroll
          for (int w = 8; w >= 1; w >>= 1) {  // keep w groups; partner = lane ^ 2w
            const bool hi = (lane & (2u * (uint32_t)w)) != 0u;
#pragma unroll
            for (int i = 0; i < w; ++i) {
              const float keep = hi ? x[i + w] : x[i];
              const float send = hi ? x[i] : x[i + w];
              x[i] = keep + __shfl_xor_sync(0xffffffffu, send, 2 * w);
            }
          }
          float sv = x[0] + __shfl_xor_sync(0xffffffffu, x[0], 1);
          sv = combine(sv, (lane & 1u) == 0u, lane >> 1);  // a query of QW warps: add its warps' sums
          sv += 0.0f;  // canonical +0
          if (part != 0) continue;
          // lane pair (2g, 2g + 1) holds group g; its even lane speaks for it when a chunk starts there
          // (start bits are also set past n_rows, so mask them to the groups in use)
          const uint32_t starts = gstart & (n_grp >= 16 ? 0xFFFFu : ((1u << n_grp) - 1u));
          const uint32_t gl = (lane >> 1) & 15u;
          const bool speaker = ((starts >> gl) & 1u) != 0u && (lane & 1u) == 0u;
          const int32_t chunk_l = (int32_t)__shfl_sync(0xffffffffu, rec, 16 + __popc(gstart & ((1u << gl) - 1u)));
          if (speaker)
            HIPER_DASSERT(chunk_l >= 0 && (MODE != 0 || chunk_l < args.score_ld), chunk_l, args.score_ld);
          if constexpr (MODE == 0) {
            if (speaker && q < args.n_q) args.scores[(int64_t)q * args.score_ld + chunk_l] = sv;
          } else {
            // top-k: a score pre-filter against the list threshold, exact key test and insert for
            // the rare rest (ascending group order)
            const uint32_t thr_hi = (uint32_t)(topk.thresh >> 32);
            uint32_t cand = __ballot_sync(0xffffffffu, speaker && float_orderable(sv) >= thr_hi);
            while (cand != 0u) {
              const int src = __ffs(cand) - 1;
              cand &= cand - 1u;
              const float s_src = __shfl_sync(0xffffffffu, sv, src);
              const int32_t c_src = __shfl_sync(0xffffffffu, chunk_l, src);
              const uint64_t key = make_key(s_src, args.id_base + c_src);
              if (key > topk.thresh) topk.insert(key, args.k, lane);
            }
          }
        }
      } else {
      int32_t ld_next = (first < c1) ? __ldg(args.d_lens + first) : 0;
      for (int64_t c = first; c < c1; c += 2, ++mine) {
        const int32_t ld = ld_next;
        if (c + 2 < c1) ld_next = __ldg(args.d_lens + c + 2);
        float m4[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
        int ix4[4] = {0, 0, 0, 0};
#pragma unroll
        for (int h = 0; h < H; ++h) {
          long long e0 = (STATS && args.stats) ? clock64() : 0;
          mbar_wait(bar_tfull(H == 1 ? grp : (uint32_t)h + 2u * grp), mine & 1u);
          long long e1 = (STATS && args.stats) ? clock64() : 0;
          if (STATS && args.stats) st_ewait_g += e1 - e0;
          tc_fence_after();
          // real columns of this half (H = 1: the chunk's length)
          const int32_t lh = H == 1 ? ld : min(max(ld - 256 * h, 0), 256);
          const uint32_t taddr = H == 1 ? taddr_base : lanes + (uint32_t)h * kAccStride;
          // early release: the accumulator goes back to the MMA as soon as its last block is in
          // registers, before that block's arithmetic (the release is on the MMA's critical path:
          // commit -> epilogue wake -> drain -> arrive -> MMA wake; args.late_release: A/B only)
          bool released = false;
          const uint32_t rel_bar = H == 1 ? tempty_leader : mapa_shared(bar_tempty(h), 0);
          for (int32_t col = 0; col < ((DBG == 1 || DBG == 2 || DBG == 4) ? 0 : lh); col += 64) {
            uint32_t v[64];
            tmem_ld64_wait(taddr + (uint32_t)col, v);
            const int rem = lh - col;
            if (rem <= 64 && !args.late_release) {  // warp-uniform: the chunk's length
              tc_fence_before();
              __syncwarp();
              if (lane == 0) mbar_arrive_cluster(rel_bar);
              released = true;
            }
            if constexpr (MODE == 2) {
              max64_arg1(v, m4[0], ix4[0], col, rem);  // chains 1..3 stay at -inf
            } else {
              if (rem >= 64) max64(v, m4);
              else max64_masked(v, m4, rem);
            }
          }
          if (!released) {
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive_cluster(rel_bar);
          }
          if (STATS && args.stats) {
            st_drain_g += clock64() - e1;
            ++st_tiles_g;
          }
        }
        const float m = fmaxf(fmaxf(m4[0], m4[1]), fmaxf(m4[2], m4[3]));
        if constexpr (MODE == 2) {
          if (q < args.n_q)
            args.amax[((int64_t)q * args.score_ld + c) * 32 + lane] = (uint8_t)ix4[0];
        }
        float sv = tok_real ? m : 0.0f;
#pragma unroll
        for (int o = 16; o >= 1; o >>= 1) sv += __shfl_xor_sync(0xffffffffu, sv, o);
        sv = combine(sv, lane == 0u, 0u);  // a query of QW warps: add its warps' sums in warp order
        sv += 0.0f;  // canonical +0
        if (part != 0) continue;
        if constexpr (MODE == 0 || MODE == 2) {
          if (lane == 0 && q < args.n_q) args.scores[(int64_t)q * args.score_ld + c] = sv;
        } else {
          // (QW > 1: only lane 0 holds the combined sum)
          const uint64_t key = make_key(QW == 1 ? sv : __shfl_sync(0xffffffffu, sv, 0), args.id_base + c);
          if (key > topk.thresh) topk.insert(key, args.k, lane);
        }
      }
      }  // !PACKED
      if constexpr (MODE == 1) {
        HIPER_DASSERT(q < args.q_pad && p < args.n_parts, q, p);
        if (part == 0) {  // partial lists: [P][kEpiGroups][q_pad][k]
          uint64_t* dst = args.partial + (((int64_t)p * kEpiGroups + grp) * args.q_pad + q) * args.k;
#pragma unroll
          for (int r = 0; r < KR; ++r) {
            const int i = r * 32 + (int)lane;
            if (i < args.k) dst[i] = topk.v[r];
          }
        }
      }
    }
  }

  if (STATS && warp < 8 && args.stats && lane == 0) {
    atomicAdd(args.stats + 3, (unsigned long long)st_drain_g);
    atomicAdd(args.stats + 4, (unsigned long long)st_ewait_g);
    atomicAdd(args.stats + 5, (unsigned long long)st_tiles_g);
  }
  // teardown: every multicast commit / remote arrive has landed before either CTA exits
  tc_fence_before();
  cluster_sync();
  if (warp == kPairAllocWarp) {
    tc_fence_after();
    tmem_dealloc_pair(tmem_base, kTmemCols);
  }
}

}  // namespace hiper
