// pooled_sm100_pair.cuh -- step a12: the pooled single-vector limit case (BASELINE.json configs[4]).
//
// With one token per query and per chunk (Lq = Ld = 1) MaxSim reduces to the dot of NORM'd vectors,
// i.e. cosine similarity of pooled embeddings -- the paper's deployed retrieval ("cosine similarity
// on the pooled embeddings"; "ranked according to the cosine similarity").
// The work is then a plain dense GEMM S = Q C^T (K = dim, e.g. 768) with a fused per-query top-k:
//  * a CTA pair (cta_group::2) computes 256 queries x 256 chunks per accumulator (M = 256, N = 256),
//    K-pipelined: every stage holds one 64-dim K-block of this CTA's 128 query rows (A) and of its
//    128 chunk rows (B), both TMA-loaded (OOB rows zero-filled: no padding in HBM);
//  * two TMEM accumulators (2 x 256 columns) alternate between the two epilogue warpgroups;
//  * epilogue thread = one query (its TMEM lane); it scans its 256 scores per tile with a float
//    threshold test and keeps a register-resident sorted top-k (KP slots) of sortable keys, written
//    to partial[p][group][q][k] at the end of the unit; topk_merge.cuh merges partitions / ranks.
//  * MODE 0 writes the dense score matrix instead (test support).
#pragma once
#include "maxsim_sm100_pair.cuh"

namespace hiper {

struct PooledArgs {
  int32_t n_q;        // real queries
  int32_t n_qtiles;   // ceil(n_q / 256)
  int32_t n_ctiles;   // ceil(n_chunks / 256)
  int32_t n_parts;    // P (partitions of chunk tiles)
  int32_t num_kb;     // dim / 64
  int32_t k;          // top-k (MODE 1), k <= KP
  int32_t n_stages;
  uint32_t stage_bytes;  // per CTA: A 128x64 + B 128x64 bf16 = 32 KiB
  int32_t q_pad;      // n_qtiles * 256 (partial row stride)
  int64_t n_chunks;
  int64_t id_base;
  float* scores;      // MODE 0: [n_q][score_ld]
  int64_t score_ld;
  uint64_t* partial;  // MODE 1: [P][kEpiGroups][q_pad][k]
  uint32_t* progress; // [n_pairs] L2 lockstep words (see maxsim_sm100_pair.cuh), or nullptr
  int32_t window;     // chunk tiles a pair may run ahead of the slowest pair
  // Shared pruning bound per query (MODE 1; nullptr = off): gthr[q] = max over every partial list of
  // query q of that list's k-th best key.  Each list holds k distinct items of a disjoint partition,
  // so no item with a key <= gthr[q] can be in the final top-k: the lists skip such items.  Without
  // it each list pays ~k(1 + ln(n/k)) insertions for its own n items (~0.5 per thread per tile here).
  unsigned long long* gthr;
  // KP == 0: a stronger shared bound.  pub8[q][p] = the 8th-best key unit (., p) holds for query q
  // (atomicMax, monotone).  If m = ceil(k / 8) partitions each hold 8 keys >= T, at least k keys of the
  // corpus are >= T, so a key below the m-th largest pub8 value cannot be in the top k.
  unsigned long long* pub8;
  // KP < 0 (APPEND, 16 < k <= 128): a per-query key bound T_q = cand_thr[q * thr_stride] (the k-th
  // best key of a corpus sample, so at least k corpus keys are >= T_q); every key >= T_q is appended
  // to the segment of (query q, partition p, group g): cand[(q * P + p) * 2 + g][0 .. cand_cap), owned
  // by that unit's thread (no atomics); cand_cnt[(q * P + p) * 2 + g] = its count, also past the
  // capacity (the host then reruns on the heap path).
  uint64_t* cand;
  uint32_t* cand_cnt;
  int32_t cand_cap;
  const uint64_t* cand_thr;
  int32_t thr_stride;
  unsigned long long* stats;  // pipeline statistics (HIPER_PIPE_STATS), or nullptr: [0] MMA cycles
                              // waiting for a free accumulator, [1] for a full stage, [2] MMA
                              // thread total, [3] epilogue drain cycles, [4] epilogue wait, [5] tiles
};

// Per-thread register top-k: the epilogue thread of query q keeps KP sortable keys in registers.
// Scanning a 64-column TMEM block is one float compare per column against the k-th score; the rare
// hits are collected in a bit mask and inserted out of the unrolled loop (a local copy of the block
// is made only then), so the insertion code exists once and the 64 scores stay in registers.
__device__ __forceinline__ float pooled_thr_score(uint64_t thr) {
  if (thr == 0ull) return -INFINITY;
  const uint32_t o = (uint32_t)(thr >> 32);
  return __uint_as_float((o & 0x80000000u) ? (o & 0x7FFFFFFFu) : ~o);
}

// DBG (ablation builds only, HIPER_DEBUG_MODE): 1 = the epilogue only waits/releases the
// accumulator (no TMEM reads, no top-k); 2 = additionally no TMA after the first stage fill;
// 3 = the epilogue reads TMEM but does no arithmetic; 4 = arithmetic without TMEM reads.
// CL = CTAs per cluster.  CL == 2: one CTA pair per cluster.  CL == 4: two pairs that score two
// query tiles (2qq, 2qq + 1) against the same chunk tiles; each chunk-tile K-block half (128 rows)
// needed by CTA r of both pairs is loaded once, half by each of them, and TMA-multicast to both, so
// the chunk operand costs half the L2 reads.  tmap_c then has a 64-row box.
// STATS: HIPER_PIPE_STATS instrumentation compiled in (diagnostics only; see the MaxSim pair kernel).
// KP > 0: each epilogue thread keeps its query's list in KP registers (k <= KP, the fast path).
// KP < 0 (APPEND): no list at all -- a key that reaches the query's sample bound T_q is appended to
// its global candidate buffer (one L2 atomic per candidate, ~32 k per query with a 1/32 sample);
// cand_select_kernel takes the exact top-k from the buffer.  The tile scan is the fast path's
// (block max, one compare) without the list upkeep, and no shared memory goes to heaps.
// KP == 0 (16 < k <= 128): each query's (unit) list is a binary MIN-heap of k keys in shared memory
// (root = the k-th best key so far = the filter threshold; empty slots are key 0, below every real key),
// so an insertion is one root replacement and a log2(k)-level sift-down by the thread that owns the
// query -- no warp-wide work, no global round trip.  The two epilogue groups serve the same 128
// queries of a unit (alternate chunk tiles), so each heap has a shared-memory spin lock; at the end of
// the unit group 0 writes the heaps (unsorted: the merge kernel needs no order) to `partial` and
// clears them, between two named barriers of the 256 epilogue threads.
template <int MODE, int KP, int DBG = 0, int CL = 2, bool STATS = false>
__global__ void __launch_bounds__(kMaxsimThreads, 1)
    pooled_sm100_pair_kernel(const __grid_constant__ CUtensorMap tmap_q,
                             const __grid_constant__ CUtensorMap tmap_c, const PooledArgs args) {
  extern __shared__ uint8_t smem_raw[];
  using namespace ptx;
  const uint32_t warp = warp_id();
  const uint32_t lane = lane_id();
  const uint32_t crank = cluster_ctarank();
  const uint32_t rank = crank & 1u;      // CTA within its pair (0 = pair leader)
  const uint32_t lead = crank & ~1u;     // cluster rank of this pair's leader
  const uint32_t p2 = crank >> 1;        // pair within the cluster
  const uint32_t pair = cluster_id_x() * (CL / 2) + p2;
  const uint32_t n_pairs = nclusters_x() * (CL / 2);
  const uint16_t pair_mask = (uint16_t)(3u << lead);
  const uint16_t all_mask = (uint16_t)((1u << CL) - 1u);

  const uint32_t base = (smem_u32(smem_raw) + 1023u) & ~1023u;
  const uint32_t sStage = base;  // n_stages x {A 16 KiB | B 16 KiB}
  const uint32_t sBar = sStage + args.n_stages * args.stage_bytes;
  const int S = args.n_stages;
  auto bar_full = [&](int s) { return sBar + 8u * s; };
  auto bar_empty = [&](int s) { return sBar + 8u * (S + s); };
  auto bar_tfull = [&](int b) { return sBar + 8u * (2 * S + b); };
  auto bar_tempty = [&](int b) { return sBar + 8u * (2 * S + 2 + b); };
  const uint32_t sTmemPtr = sBar + 8u * (2 * S + 4);
  // KP == 0: [128 queries][k | 1] u64 min-heaps (odd stride: conflict-free 64-bit banks) + 128 locks
  const uint32_t kst = (uint32_t)args.k | 1u;
  volatile uint64_t* heaps = reinterpret_cast<volatile uint64_t*>(smem_raw + (sBar + 1024u - smem_u32(smem_raw)));
  uint32_t* hlocks = reinterpret_cast<uint32_t*>(smem_raw + (sBar + 1024u + 128u * kst * 8u - smem_u32(smem_raw)));
  // KP == 0: [128 queries][8] u64, each query's 8 best keys of the unit (descending), under the lock
  volatile uint64_t* top8 = reinterpret_cast<volatile uint64_t*>(
      smem_raw + (sBar + 1024u + 128u * kst * 8u + 512u - smem_u32(smem_raw)));
  uint32_t* tmem_ptr_generic =
      reinterpret_cast<uint32_t*>(smem_raw + (sTmemPtr - smem_u32(smem_raw)));

  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(bar_full(s), 1);
      mbar_init(bar_empty(s), CL / 2);  // every pair whose operands this stage (also) holds
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

  // units: (query tile, partition) for CL == 2; (query-tile pair, partition) for CL == 4, the two
  // pairs of a cluster taking query tiles 2qq and 2qq + 1 of the same unit
  const int32_t n_qu = args.n_qtiles / (CL / 2);
  const int32_t n_units = n_qu * args.n_parts;
  const uint32_t ustride = n_pairs / (CL / 2);  // clusters
  const uint32_t ufirst = pair / (CL / 2);
  auto decode = [&](int32_t u, int32_t& qt, int32_t& p, int32_t& t0, int32_t& t1) {
    p = u / n_qu;
    qt = (u - p * n_qu) * (CL / 2) + (int32_t)p2;
    t0 = (int32_t)((int64_t)p * args.n_ctiles / args.n_parts);
    t1 = (int32_t)((int64_t)(p + 1) * args.n_ctiles / args.n_parts);
  };

  if (warp == kPairProducerWarp) {
    if (lane == 0) {
      prefetch_tmap(&tmap_q);
      prefetch_tmap(&tmap_c);
      int s = 0;
      uint32_t ph = 0, it = 0, streamed = 0;  // streamed: chunk tiles of this pair's finished units
      for (int32_t u = (int32_t)ufirst; u < n_units; u += (int32_t)ustride, ++it) {
        int32_t qt, p, t0, t1;
        decode(u, qt, p, t0, t1);
        for (int32_t ct = t0; ct < t1; ++ct) {
          if (args.progress != nullptr && rank == 0 && ((ct - t0) & 3) == 0) {
            const uint32_t pos = streamed + (uint32_t)(ct - t0);  // continuous across units
            lockstep_publish(args.progress, pair, pos);
            lockstep_wait(args.progress, n_pairs, pos, (uint32_t)args.window);
          }
          for (int kb = 0; kb < args.num_kb; ++kb) {
            mbar_wait(bar_empty(s), ph ^ 1u);
            if (DBG == 2 && (it > 0 || ct - t0 >= 1)) {
              if (rank == 0) mbar_arrive(bar_full(s));
              if (++s == S) { s = 0; ph ^= 1u; }
              continue;
            }
            if (rank == 0) mbar_arrive_expect_tx(bar_full(s), 2u * args.stage_bytes);
            const uint32_t full_leader = mapa_shared(bar_full(s), lead);
            const uint32_t st = sStage + s * args.stage_bytes;
            tma_load_2d_pair(st, &tmap_q, full_leader, kb * 64, qt * 256 + (int32_t)rank * 128);
            if constexpr (CL == 2) {
              tma_load_2d_pair(st + 16384u, &tmap_c, full_leader, kb * 64, ct * 256 + (int32_t)rank * 128);
            } else {  // my 64-row half of the 128 chunk rows CTA `rank` of both pairs needs
              tma_load_2d_pair_mc(st + 16384u + p2 * 8192u, &tmap_c, full_leader, kb * 64,
                                  ct * 256 + (int32_t)rank * 128 + (int32_t)p2 * 64,
                                  (uint16_t)((1u << rank) | (1u << (2u + rank))));
            }
            if (++s == S) { s = 0; ph ^= 1u; }
          }
        }
        streamed += (uint32_t)(t1 - t0);
      }
      if (args.progress != nullptr && rank == 0) lockstep_publish(args.progress, pair, 0xFFFFFFFFu);
    }
  } else if (warp == kPairMmaWarp) {
    if (rank == 0 && lane == 0) {
      const uint32_t idesc = idesc_bf16_f32(256, 256);
      int s = 0;
      uint32_t ph = 0, t = 0;
      long long st_acc = 0, st_full = 0;
      const long long st_t0 = clock64();
      for (int32_t u = (int32_t)ufirst; u < n_units; u += (int32_t)ustride) {
        int32_t qt, p, t0, t1;
        decode(u, qt, p, t0, t1);
        for (int32_t ct = t0; ct < t1; ++ct, ++t) {
          const uint32_t acc = t & 1u, tph = (t >> 1) & 1u;
          long long w0 = (STATS && args.stats) ? clock64() : 0;
          mbar_wait(bar_tempty(acc), tph ^ 1u);
          if (STATS && args.stats) st_acc += clock64() - w0;
          tc_fence_after();
          const uint32_t d_tmem = tmem_base + acc * kAccStride;
          for (int kb = 0; kb < args.num_kb; ++kb) {
            if (STATS && args.stats) w0 = clock64();
            mbar_wait(bar_full(s), ph);
            if (STATS && args.stats) st_full += clock64() - w0;
            tc_fence_after();
            const uint32_t st = sStage + s * args.stage_bytes;
#pragma unroll
            for (int kk = 0; kk < 4; ++kk)
              mma_bf16_ss_pair(d_tmem, umma_desc_sw128(st + kk * 32),
                               umma_desc_sw128(st + 16384u + kk * 32), idesc,
                               (kb | kk) != 0 ? 1u : 0u);
            mma_commit_pair_mc(bar_empty(s), all_mask);  // every CTA that wrote into this stage
            if (++s == S) { s = 0; ph ^= 1u; }
          }
          mma_commit_pair_mc(bar_tfull(acc), pair_mask);
        }
      }
      if (STATS && args.stats) {
        atomicAdd(args.stats + 0, (unsigned long long)st_acc);
        atomicAdd(args.stats + 1, (unsigned long long)st_full);
        atomicAdd(args.stats + 2, (unsigned long long)(clock64() - st_t0));
      }
    }
  } else if (warp < 8) {
    const uint32_t qslot = warp & 3u;
    const uint32_t grp = warp >> 2;
    const uint32_t taddr_base = tmem_base + ((qslot * 32u) << 16) + grp * kAccStride;
    const uint32_t tempty_leader = mapa_shared(bar_tempty(grp), lead);
    const int32_t k = args.k;
    uint32_t t = 0, mine = 0;
    long long st_drain = 0, st_ewait = 0, st_tiles = 0, st_any = 0, st_ins = 0, st_cs = 0, st_spin = 0,
              st_csc = 0;
    if constexpr (MODE == 1 && KP == 0) {  // empty heaps (key 0) and free locks before the first unit
      if (grp == 0) {
        const uint32_t qi0 = qslot * 32u + lane;
        for (int m = 0; m < k; ++m) heaps[qi0 * kst + m] = 0ull;
        for (int m = 0; m < 8; ++m) top8[qi0 * 8 + m] = 0ull;
        hlocks[qi0] = 0u;
      }
      named_bar_sync(9, 256);
    }
    // KP == 0: T = the m-th largest of the partitions' published 8th-best keys of query qq,
    // m = ceil(k / 8) (a running descending list of the 16 largest)
    auto pub8_bound = [&](int32_t qq) -> uint64_t {
      const int m8 = (k + 7) >> 3;
      uint64_t best[16];
#pragma unroll
      for (int x = 0; x < 16; ++x) best[x] = 0ull;
      const volatile unsigned long long* row = args.pub8 + (int64_t)qq * args.n_parts;
      for (int32_t pp = 0; pp < args.n_parts; ++pp) {
        uint64_t val = row[pp];
#pragma unroll
        for (int x = 0; x < 16; ++x) {
          const uint64_t hi = best[x] > val ? best[x] : val;
          val = best[x] > val ? val : best[x];
          best[x] = hi;
        }
      }
      uint64_t T = 0ull;
#pragma unroll
      for (int x = 0; x < 16; ++x)
        if (x == m8 - 1) T = best[x];
      return T;
    };
    for (int32_t u = (int32_t)ufirst; u < n_units; u += (int32_t)ustride) {
      int32_t qt, p, t0, t1;
      decode(u, qt, p, t0, t1);
      const int32_t q = qt * 256 + (int32_t)rank * 128 + (int32_t)qslot * 32 + (int32_t)lane;
      uint64_t v[KP > 0 ? KP : 1];
#pragma unroll
      for (int m = 0; m < (KP > 0 ? KP : 1); ++m) v[m] = 0ull;
      const uint32_t qi = qslot * 32u + lane;  // this thread's query within the CTA (its heap)
      volatile uint64_t* heap = heaps + qi * kst;
      uint64_t thr = 0ull;        // key of rank k-1 (0 while the list is not full)
      uint64_t gth = 0ull, pub = 0ull;  // shared bound seen / own thr last published
      if (args.gthr != nullptr && q < args.q_pad)
        gth = *reinterpret_cast<volatile unsigned long long*>(args.gthr + q);
      if constexpr (KP == 0) {
        if (args.pub8 != nullptr && q < args.q_pad) {
          const uint64_t T = pub8_bound(q);
          gth = T > gth ? T : gth;
        }
      }
      if constexpr (KP < 0)  // APPEND: the static sample bound (a real key: its chunk is appended too)
        gth = (q < args.n_q) ? args.cand_thr[(int64_t)q * args.thr_stride] : ~0ull;
      uint32_t n_app = 0;  // APPEND: keys this thread appended to its (q, p, grp) segment
      uint64_t* seg = args.cand + (((int64_t)q * args.n_parts + p) * kEpiGroups + grp) * args.cand_cap;
      uint64_t lim = gth;         // max(thr, gth): only keys above it can enter
      const uint32_t mine0 = mine;  // this unit's first tile (KP == 0: refresh the bound often early)
      float thr_f = pooled_thr_score(lim);  // its score: most candidates fail one float compare
      const int32_t first = t0 + (int32_t)((grp - (t & 1u)) & 1u);
      t += (uint32_t)(t1 - t0);
      for (int32_t ct = first; ct < t1; ct += 2, ++mine) {
        long long e0 = (STATS && args.stats) ? clock64() : 0;
        mbar_wait(bar_tfull(grp), mine & 1u);
        long long e1 = (STATS && args.stats) ? clock64() : 0;
        if (STATS && args.stats) st_ewait += e1 - e0;
        tc_fence_after();
        const int64_t cbase = (int64_t)ct * 256;
        const int64_t left = args.n_chunks - cbase;
        const int32_t ncols = (DBG == 1 || DBG == 2) ? 0 : (left < 256 ? (int32_t)left : 256);
        for (int32_t col = 0; col < ncols; col += 64) {
          uint32_t r[64];
          if constexpr (DBG == 4) {  // ablation: no TMEM read, compute on fixed data
#pragma unroll
            for (int j = 0; j < 64; ++j) r[j] = __float_as_uint(-1.0f - (float)j);
          } else {
            tmem_ld64_wait(taddr_base + (uint32_t)col, r);
          }
          if constexpr (DBG == 3) continue;  // ablation: TMEM read only
          if constexpr (MODE == 0) {
            if (q < args.n_q) {
              float* dst = args.scores + (int64_t)q * args.score_ld + cbase + col;
#pragma unroll
              for (int j = 0; j < 64; ++j)
                if (col + j < ncols) dst[j] = __uint_as_float(r[j]) + 0.0f;
            }
          } else {
            const int32_t nj = ncols - col;  // >= 64 except in the corpus' last tile
            // common case first: one max over the block (21 FMNMX3) and a single compare; the
            // per-column hit mask is built only when some column can enter the list
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
              if (STATS && args.stats) ++st_any;
#pragma unroll
              for (int j = 0; j < 64; ++j)
                hits |= (uint64_t)(__uint_as_float(r[j]) >= thr_f && j < nj) << j;
            }
            if constexpr (KP < 0) {
              if (hits) {  // rare: append the keys >= T_q (exact key test past the float filter)
                float xs[64];
#pragma unroll
                for (int jj = 0; jj < 64; ++jj) xs[jj] = __uint_as_float(r[jj]) + 0.0f;
                while (hits) {
                  const int j = __ffsll((long long)hits) - 1;
                  hits &= hits - 1;
                  const uint64_t key = make_key(xs[j], args.id_base + cbase + col + j);
                  if (key >= gth) {
                    if (STATS && args.stats) ++st_ins;
                    if (n_app < (uint32_t)args.cand_cap) seg[n_app] = key;
                    ++n_app;
                  }
                }
              }
            } else if constexpr (KP == 0) {
              if (hits) {  // rare: this thread's query heap, under its lock (shared with the other group)
                float xs[64];
#pragma unroll
                for (int jj = 0; jj < 64; ++jj) xs[jj] = __uint_as_float(r[jj]) + 0.0f;
                long long cs0 = (STATS && args.stats) ? clock64() : 0;
                while (atomicCAS_block(hlocks + qi, 0u, 1u) != 0u) {
                }
                __threadfence_block();
                if (STATS && args.stats) {
                  st_spin += clock64() - cs0;
                  ++st_cs;
                }
                uint64_t root = heap[0];
                while (hits) {
                  const int j = __ffsll((long long)hits) - 1;
                  hits &= hits - 1;
                  const uint64_t key = make_key(xs[j], args.id_base + cbase + col + j);
                  if (key > root && key > gth) {
                    if (STATS && args.stats) ++st_ins;
                    uint32_t i = 0;  // sift the new key down from the root
                    while (true) {
                      const uint32_t l = 2u * i + 1u;
                      if (l >= (uint32_t)k) break;
                      uint64_t cv = heap[l];
                      uint32_t c = l;
                      if (l + 1u < (uint32_t)k) {
                        const uint64_t rv = heap[l + 1u];
                        if (rv < cv) {
                          cv = rv;
                          c = l + 1u;
                        }
                      }
                      if (cv >= key) break;
                      heap[i] = cv;
                      i = c;
                    }
                    heap[i] = key;
                    root = heap[0];
                    if (args.pub8 != nullptr) {  // the unit's 8 best keys of this query
                      volatile uint64_t* t8 = top8 + qi * 8;
                      if (key > t8[7]) {
                        int pos = 7;
                        while (pos > 0 && t8[pos - 1] < key) {
                          t8[pos] = t8[pos - 1];
                          --pos;
                        }
                        t8[pos] = key;
                      }
                    }
                  }
                }
                const uint64_t my8 = args.pub8 != nullptr ? top8[qi * 8 + 7] : 0ull;
                __threadfence_block();
                atomicExch_block(hlocks + qi, 0u);
                if (my8 != 0ull && q < args.q_pad)
                  atomicMax(args.pub8 + (int64_t)q * args.n_parts + p, (unsigned long long)my8);
                thr = root;
                lim = thr > gth ? thr : gth;
                thr_f = pooled_thr_score(lim);
              }
            } else if (hits) {
              float xs[64];  // rare path: a local copy so the hits can be indexed dynamically
#pragma unroll
              for (int j = 0; j < 64; ++j) xs[j] = __uint_as_float(r[j]) + 0.0f;
              while (hits) {
                const int j = __ffsll((long long)hits) - 1;
                hits &= hits - 1;
                uint64_t key = make_key(xs[j], args.id_base + cbase + col + j);
                if (key > lim) {
                  if (STATS && args.stats) ++st_ins;
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
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive_cluster(tempty_leader);
        if (STATS && args.stats) {
          st_drain += clock64() - e1;
          ++st_tiles;
        }
        if constexpr (MODE == 1 && KP >= 0) {
          if (args.gthr != nullptr && q < args.q_pad) {
            if (thr > pub) {  // publish this list's k-th key; learn the others'
              const uint64_t old = atomicMax(args.gthr + q, (unsigned long long)thr);
              pub = thr;
              gth = old > gth ? old : gth;
            } else if ((mine & (KP == 0 ? 1u : 7u)) == 0) {
              const uint64_t cur = *reinterpret_cast<volatile unsigned long long*>(args.gthr + q);
              gth = cur > gth ? cur : gth;
            }
            if constexpr (KP == 0) {
              // every tile during the unit's first 8 (the bound rises fastest while the heaps fill),
              // then every 8th
              if (args.pub8 != nullptr && (mine - mine0 < 8u || (mine & 7u) == 0)) {
                const uint64_t T = pub8_bound(q);
                gth = T > gth ? T : gth;
              }
            }
            const uint64_t nl = thr > gth ? thr : gth;
            if (nl != lim) {
              lim = nl;
              thr_f = pooled_thr_score(lim);
            }
          }
        }
      }
      if constexpr (MODE == 1 && KP < 0) {
        if (q < args.n_q) args.cand_cnt[((int64_t)q * args.n_parts + p) * kEpiGroups + grp] = n_app;
      }
      if constexpr (MODE == 1 && KP > 0) {
        if (q < args.n_q) {
          uint64_t* dst = args.partial + (((int64_t)p * kEpiGroups + grp) * args.q_pad + q) * k;
#pragma unroll
          for (int m = 0; m < KP; ++m)
            if (m < k) dst[m] = v[m];
        }
      }
      if constexpr (MODE == 1 && KP == 0) {
        named_bar_sync(9, 256);  // both groups are done with this unit's heaps
        if (grp == 0) {           // the unit's list of query q (slot grp 0 of the partial layout)
          uint64_t* dst = args.partial + ((int64_t)p * kEpiGroups * args.q_pad + q) * k;
          for (int m = 0; m < k; ++m) {
            if (q < args.n_q) dst[m] = heap[m];
            heap[m] = 0ull;
          }
          for (int m = 0; m < 8; ++m) top8[qi * 8 + m] = 0ull;
        }
        named_bar_sync(9, 256);  // cleared before the next unit's first insertion
      }
    }
    if (STATS && args.stats && lane == 0) {
      atomicAdd(args.stats + 3, (unsigned long long)st_drain);
      atomicAdd(args.stats + 4, (unsigned long long)st_ewait);
      atomicAdd(args.stats + 5, (unsigned long long)st_tiles);
    }
    if (STATS && args.stats) {
      atomicAdd(args.stats + 6, (unsigned long long)st_any);
      atomicAdd(args.stats + 7, (unsigned long long)st_ins);
      if (lane == 0) {
        atomicAdd(args.stats + 8, (unsigned long long)st_cs);
        atomicAdd(args.stats + 9, (unsigned long long)st_spin);
        atomicAdd(args.stats + 10, (unsigned long long)st_csc);
      }
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
