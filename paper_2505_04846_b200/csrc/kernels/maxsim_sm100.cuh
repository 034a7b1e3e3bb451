// maxsim_sm100.cuh -- steps a3-a6: the fused MaxSim kernel (TMA -> tcgen05.mma -> TMEM -> epilogue).
//
//   S(q, c) = sum_{i < len_q} max_{j < len_c} < q_i , d_{c,j} >       (§2.2, Fig.3B
//                                                                    PAPER.md:228)
//
// Work decomposition:
//  * A "row group" g = 4 queries x 32 padded query-token rows = the M = 128 rows of one tcgen05.mma.
//    Its A tile (128 rows x dim bf16, K-major, 128B-swizzled) stays resident in shared memory for a
//    whole unit (double-buffered across units).
//  * The corpus is cut into P contiguous partitions; a unit = (row group g, partition p).  Units are
//    ordered partition-major and dealt round-robin to a persistent grid (one CTA per SM), so the CTAs
//    of one wave stream the same chunk tiles at the same time and HBM sees each tile ~once (L2 reuse).
//  * Per chunk: TMA brings the chunk's ld_pad token rows (64 dims per box, 128B swizzle) into a
//    pipeline stage; one elected thread issues dim/16 tcgen05.mma (M=128, N=ld_pad, K=16) into one of
//    two TMEM accumulators (128 lanes x 256 fp32 columns each = all 512 TMEM columns), so the epilogue
//    of chunk t overlaps the MMAs of chunk t+1.
//  * Epilogue warps 4..7: warp w reads TMEM lanes 32*(w%4)..+31 = the 32 token rows of query slot w%4;
//    each thread (one query token i) reduces max over the chunk's real columns j < len_c (columns
//    >= len_c are never read: reading R2), the warp then sums over real query tokens i < len_q
//    (butterfly shuffle, fixed order: R3).  The q x d token-similarity tensor never leaves TMEM.
//  * MODE 0 writes S[q][c] (dense scores: ColTrast in-batch matrix a10, test export).
//    MODE 1 keeps a per-(unit, query) top-k in registers (KR x 32 lanes, sortable 64-bit keys
//    (orderable(score) << 32 | ~id): larger key = higher score, then lower id -- reading R6) and writes
//    it to partial[p][q][0..k) at the end of the unit (a6); topk_merge.cuh merges partitions (a7).
#pragma once
#include <cuda.h>
#include <cuda_bf16.h>
#include <cstdint>

#include "../ptx.cuh"

namespace hiper {

struct MaxsimArgs {
  int32_t n_q;       // real queries
  int32_t n_groups;  // G = ceil(n_q / 4)
  int32_t n_parts;   // P
  int32_t ld_pad;    // MMA N = token rows per chunk tile (multiple of 16, <= 256)
  int32_t num_kb;    // dim / 64
  int32_t k;         // top-k (MODE 1)
  int32_t n_stages;  // B pipeline stages
  uint32_t a_bytes;  // one A buffer (num_kb * 16 KiB)
  uint32_t stage_bytes;  // ld_pad * 128
  int64_t n_chunks;
  int64_t id_base;
  const int32_t* q_lens;  // device [n_q]
  const int32_t* d_lens;  // device [n_chunks]
  float* scores;          // MODE 0: [n_q][score_ld]
  int64_t score_ld;
  uint64_t* partial;      // MODE 1: [P][4G][k]
  uint32_t* progress;     // pair kernel: [n_pairs] progress words for L2 lockstep, or nullptr
  uint8_t* amax;          // MODE 2: [n_q][score_ld][32] argmax doc-token index of every max
  const int32_t* cand;    // rerank (N3): [G][n_chunks] chunk index per slot of each row group
                          // (-1 = empty slot), or nullptr = the corpus itself
  int32_t window;         // chunks a pair may run ahead of the slowest pair (lockstep window)
  const int64_t* row_of;  // rerank over a packed index: first packed row of each chunk (its rows are
                          // row_of[c] + j); nullptr = dense layout, chunk c at row c * ld_pad
  // packed layout (N4, PACKED kernels): slot c of the kernel is tile c of a length-bucketed packed
  // corpus, described by a 128-B record recs[c][0..32): w0 = n_rows | n_ent << 16 (n_rows a multiple
  // of 16, <= 256; n_ent <= 16 chunks), w1 = start mask (bit g: a chunk begins at column group g of
  // 16), w4 = first packed row, w16 + e = chunk index of slot e (slots in column order).  The
  // padding rows of a chunk's last 16-row group repeat its last real row (no column masking).
  const uint32_t* recs;
  unsigned long long* stats;  // HIPER_PIPE_STATS diagnostics (see pooled_sm100_pair.cuh), or nullptr
};

// warp 0 TMA, 1 MMA, 2 TMEM alloc, 3 spare; warps 4-7 = epilogue warpgroup 0 (accumulator 0, even
// chunks), warps 8-11 = epilogue warpgroup 1 (accumulator 1, odd chunks).
constexpr int kMaxsimThreads = 384;
constexpr int kEpiGroups = 2;
constexpr uint32_t kTmemCols = 512;
constexpr uint32_t kAccStride = 256;  // TMEM columns per accumulator buffer

__device__ __forceinline__ uint32_t float_orderable(float f) {
  const uint32_t b = __float_as_uint(f);
  return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}
__device__ __forceinline__ uint64_t make_key(float score, int64_t gid) {
  return ((uint64_t)float_orderable(score) << 32) | (uint64_t)(~(uint32_t)gid);
}

// Warp-resident sorted top-k list: lane l, register r holds rank r*32 + l (descending keys).
template <int KR>
struct WarpTopK {
  uint64_t v[KR];
  uint64_t thresh;  // key of rank k-1 (0 while the list is not full)

  __device__ __forceinline__ void init() {
#pragma unroll
    for (int r = 0; r < KR; ++r) v[r] = 0ull;
    thresh = 0ull;
  }
  // Warp-uniform call with a warp-uniform key > thresh.
  __device__ __forceinline__ void insert(uint64_t key, int k, uint32_t lane) {
    int pos = 0;
#pragma unroll
    for (int r = 0; r < KR; ++r) {
      const int i = r * 32 + (int)lane;
      pos += __popc(__ballot_sync(0xffffffffu, i < k && v[r] > key));
    }
#pragma unroll
    for (int r = KR - 1; r >= 0; --r) {
      uint64_t prev = __shfl_up_sync(0xffffffffu, v[r], 1);
      const uint64_t carry = (r > 0) ? __shfl_sync(0xffffffffu, v[r > 0 ? r - 1 : 0], 31) : 0ull;
      if (lane == 0) prev = carry;
      const int i = r * 32 + (int)lane;
      v[r] = (i < pos) ? v[r] : (i == pos ? key : prev);
    }
    uint64_t tv = 0ull;
#pragma unroll
    for (int r = 0; r < KR; ++r)
      if (r == ((k - 1) >> 5)) tv = v[r];
    thresh = __shfl_sync(0xffffffffu, tv, (k - 1) & 31);
  }
};

__device__ __forceinline__ void unit_decode(const MaxsimArgs& a, int32_t u, int32_t& g, int32_t& p,
                                            int64_t& c0, int64_t& c1) {
  p = u / a.n_groups;
  g = u - p * a.n_groups;
  c0 = (int64_t)p * a.n_chunks / a.n_parts;
  c1 = (int64_t)(p + 1) * a.n_chunks / a.n_parts;
}

// Running max over 64 TMEM columns with 4 independent FMNMX3 chains (ILP 4: the reduction is
// issue-bound, not latency-bound).
__device__ __forceinline__ void max64(const uint32_t (&v)[64], float (&m)[4]) {
#pragma unroll
  for (int i = 0; i < 64; i += 8) {
#pragma unroll
    for (int c = 0; c < 4; ++c)
      m[c] = fmaxf(fmaxf(m[c], __uint_as_float(v[i + 2 * c])), __uint_as_float(v[i + 2 * c + 1]));
  }
}
// Running max over N (16 or 32) columns, all real / only the first `rem` real (reading R2).
template <int N>
__device__ __forceinline__ void maxN(const uint32_t (&v)[N], float (&m)[4]) {
#pragma unroll
  for (int i = 0; i < N; i += 8) {
#pragma unroll
    for (int c = 0; c < 4; ++c)
      m[c] = fmaxf(fmaxf(m[c], __uint_as_float(v[i + 2 * c])), __uint_as_float(v[i + 2 * c + 1]));
  }
}
template <int N>
__device__ __forceinline__ void maxN_masked(const uint32_t (&v)[N], float (&m)[4], int rem) {
#pragma unroll
  for (int i = 0; i < N; ++i) {
    const float x = (i < rem) ? __uint_as_float(v[i]) : -INFINITY;
    m[i & 3] = fmaxf(m[i & 3], x);
  }
}
// Same, for a ragged tail: columns >= rem are excluded from the max (reading R2).
__device__ __forceinline__ void max64_masked(const uint32_t (&v)[64], float (&m)[4], int rem) {
#pragma unroll
  for (int i = 0; i < 64; ++i) {
    const float x = (i < rem) ? __uint_as_float(v[i]) : -INFINITY;
    m[i & 3] = fmaxf(m[i & 3], x);
  }
}
// Running max and argmax (lowest column on exact ties) with one running pair per thread: the block
// max costs 21 FMNMX3; only a block that raises the running max is scanned (downwards, == test) for
// its lowest column attaining it.  The lowest match is always a real column: the block max is
// attained by one, and padded columns (index >= rem) come after every real one.
__device__ __forceinline__ void max64_arg1(const uint32_t (&v)[64], float& m, int& ix, int base,
                                           int rem) {
  float b[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
  if (rem >= 64) max64(v, b);
  else max64_masked(v, b, rem);
  const float mb = fmaxf(fmaxf(b[0], b[1]), fmaxf(b[2], b[3]));
  if (mb > m) {
    int j = 63;
#pragma unroll
    for (int i = 63; i >= 0; --i) j = (__uint_as_float(v[i]) == mb) ? i : j;
    m = mb;
    ix = base + j;
  }
}

template <int MODE, int KR>
__global__ void __launch_bounds__(kMaxsimThreads, 1)
    maxsim_sm100_kernel(const __grid_constant__ CUtensorMap tmap_q,
                        const __grid_constant__ CUtensorMap tmap_d, const MaxsimArgs args) {
  extern __shared__ uint8_t smem_raw[];
  using namespace ptx;
  const uint32_t warp = warp_id();
  const uint32_t lane = lane_id();

  // ---- shared memory carve-up (1024-B aligned for the 128B swizzle atoms)
  const uint32_t base = (smem_u32(smem_raw) + 1023u) & ~1023u;
  const uint32_t sA = base;                                  // 2 x a_bytes
  const uint32_t sB = sA + 2 * args.a_bytes;                 // n_stages x stage_bytes
  const uint32_t sBar = sB + args.n_stages * args.stage_bytes;
  const int S = args.n_stages;
  auto bar_full = [&](int s) { return sBar + 8u * s; };
  auto bar_empty = [&](int s) { return sBar + 8u * (S + s); };
  auto bar_afull = [&](int b) { return sBar + 8u * (2 * S + b); };
  auto bar_aempty = [&](int b) { return sBar + 8u * (2 * S + 2 + b); };
  auto bar_tfull = [&](int b) { return sBar + 8u * (2 * S + 4 + b); };
  auto bar_tempty = [&](int b) { return sBar + 8u * (2 * S + 6 + b); };
  const uint32_t sTmemPtr = sBar + 8u * (2 * S + 8);
  uint32_t* tmem_ptr_generic =
      reinterpret_cast<uint32_t*>(smem_raw + (sTmemPtr - smem_u32(smem_raw)));

  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(bar_full(s), 1);
      mbar_init(bar_empty(s), 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(bar_afull(b), 1);
      mbar_init(bar_aempty(b), 1);
      mbar_init(bar_tfull(b), 1);
      mbar_init(bar_tempty(b), 4);  // the 4 warps of the epilogue group that owns buffer b
    }
    fence_mbarrier_init();
  }
  if (warp == 2) {
    tmem_alloc(sTmemPtr, kTmemCols);
    tmem_relinquish();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *reinterpret_cast<volatile uint32_t*>(tmem_ptr_generic);

  const int32_t n_units = args.n_groups * args.n_parts;

  if (warp == 0) {
    // ================= TMA producer =================
    if (lane == 0) {
      prefetch_tmap(&tmap_q);
      prefetch_tmap(&tmap_d);
      int s = 0;
      uint32_t ph = 0, it = 0;
      for (int32_t u = blockIdx.x; u < n_units; u += gridDim.x, ++it) {
        int32_t g, p;
        int64_t c0, c1;
        unit_decode(args, u, g, p, c0, c1);
        const uint32_t ab = it & 1u, aph = (it >> 1) & 1u;
        mbar_wait(bar_aempty(ab), aph ^ 1u);
        mbar_arrive_expect_tx(bar_afull(ab), args.a_bytes);
        for (int kb = 0; kb < args.num_kb; ++kb)
          tma_load_2d(sA + ab * args.a_bytes + kb * 16384u, &tmap_q, bar_afull(ab), kb * 64, g * 128);
        for (int64_t c = c0; c < c1; ++c) {
          for (int kb = 0; kb < args.num_kb; ++kb) {
            mbar_wait(bar_empty(s), ph ^ 1u);
            mbar_arrive_expect_tx(bar_full(s), args.stage_bytes);
            tma_load_2d(sB + s * args.stage_bytes, &tmap_d, bar_full(s), kb * 64,
                        (int32_t)(c * args.ld_pad));
            if (++s == S) { s = 0; ph ^= 1u; }
          }
        }
      }
    }
  } else if (warp == 1) {
    // ================= MMA issuer (single thread) =================
    if (lane == 0) {
      const uint32_t idesc = idesc_bf16_f32(128, (uint32_t)args.ld_pad);
      int s = 0;
      uint32_t ph = 0, it = 0, t = 0;
      for (int32_t u = blockIdx.x; u < n_units; u += gridDim.x, ++it) {
        int32_t g, p;
        int64_t c0, c1;
        unit_decode(args, u, g, p, c0, c1);
        const uint32_t ab = it & 1u, aph = (it >> 1) & 1u;
        mbar_wait(bar_afull(ab), aph);
        tc_fence_after();
        const uint32_t a_tile = sA + ab * args.a_bytes;
        for (int64_t c = c0; c < c1; ++c, ++t) {
          const uint32_t acc = t & 1u, tph = (t >> 1) & 1u;
          mbar_wait(bar_tempty(acc), tph ^ 1u);
          tc_fence_after();
          const uint32_t d_tmem = tmem_base + acc * kAccStride;
          for (int kb = 0; kb < args.num_kb; ++kb) {
            mbar_wait(bar_full(s), ph);
            tc_fence_after();
            const uint32_t a_kb = a_tile + kb * 16384u;
            const uint32_t b_st = sB + s * args.stage_bytes;
#pragma unroll
            for (int kk = 0; kk < 4; ++kk) {
              mma_bf16_ss(d_tmem, umma_desc_sw128(a_kb + kk * 32), umma_desc_sw128(b_st + kk * 32),
                          idesc, (kb | kk) != 0 ? 1u : 0u);
            }
            mma_commit(bar_empty(s));  // frees the stage once these MMAs have read it
            if (++s == S) { s = 0; ph ^= 1u; }
          }
          mma_commit(bar_tfull(acc));  // accumulator complete -> epilogue
        }
        mma_commit(bar_aempty(ab));  // A tile no longer needed
      }
    }
  } else if (warp >= 4) {
    // ================= epilogue: masked max over doc tokens, masked sum over query tokens ====
    // Group e owns TMEM accumulator e, i.e. the chunks with global chunk counter t % 2 == e, so each
    // group has two MMA periods per chunk to drain its accumulator.
    const uint32_t qslot = warp & 3u;
    const uint32_t grp = (warp - 4u) >> 2;
    const uint32_t taddr_base = tmem_base + ((qslot * 32u) << 16) + grp * kAccStride;
    uint32_t t = 0, mine = 0;
    for (int32_t u = blockIdx.x; u < n_units; u += gridDim.x) {
      int32_t g, p;
      int64_t c0, c1;
      unit_decode(args, u, g, p, c0, c1);
      const int32_t q = g * 4 + (int32_t)qslot;
      const int32_t lq = q < args.n_q ? __ldg(args.q_lens + q) : 0;
      WarpTopK<KR> topk;
      topk.init();
      // first chunk of this unit owned by this group
      const int64_t first = c0 + (int64_t)((grp - (t & 1u)) & 1u);
      t += (uint32_t)(c1 - c0);
      int32_t ld_next = (first < c1) ? __ldg(args.d_lens + first) : 0;
      for (int64_t c = first; c < c1; c += 2, ++mine) {
        const int32_t ld = ld_next;
        if (c + 2 < c1) ld_next = __ldg(args.d_lens + c + 2);
        mbar_wait(bar_tfull(grp), mine & 1u);
        tc_fence_after();
        float m4[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
        for (int32_t col = 0; col < ld; col += 64) {
          uint32_t v[64];
          tmem_ld64_wait(taddr_base + (uint32_t)col, v);
          const int rem = ld - col;
          if (rem >= 64) max64(v, m4);
          else max64_masked(v, m4, rem);
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(bar_tempty(grp));
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
        // partial lists: [P][kEpiGroups][4G = n_q_pad][k]
        uint64_t* dst = args.partial +
                        (((int64_t)p * kEpiGroups + grp) * args.n_groups * 4 + q) * args.k;
#pragma unroll
        for (int r = 0; r < KR; ++r) {
          const int i = r * 32 + (int)lane;
          if (i < args.k) dst[i] = topk.v[r];
        }
      }
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc(tmem_base, kTmemCols);
  }
}

}  // namespace hiper
