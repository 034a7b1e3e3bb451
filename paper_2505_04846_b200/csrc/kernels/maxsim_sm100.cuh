// maxsim_sm100.cuh -- steps a3-a6: shared definitions of the fused MaxSim kernel (TMA -> tcgen05.mma
// -> TMEM -> epilogue); the kernel itself is the CTA-pair kernel in maxsim_sm100_pair.cuh.
//
//   S(q, c) = sum_{i < len_q} max_{j < len_c} < q_i , d_{c,j} >       (§2.2, Fig.3B
//                                                                    PAPER.md:228)
//
// Work decomposition:
//  * A query occupies QS = 32 * QW padded token rows (QW = 1, 2, 4 for q_max_len <= 32, 64, 128), so
//    a CTA's M = 128 A tile holds 4 / QW queries and a CTA pair's M = 256 holds 8 / QW ("row group").
//    The A tile (128 rows x dim bf16, K-major, 128B-swizzled) stays resident in shared memory for a
//    whole unit.
//  * The corpus is cut into P contiguous partitions; a unit = (row group g, partition p).  Units are
//    ordered partition-major and dealt round-robin to a persistent grid (one CTA pair per TPC), so the
//    pairs of one wave stream the same chunk tiles at the same time and HBM sees each tile ~once.
//  * Per chunk: TMA brings the chunk's token rows (64 dims per box, 128B swizzle) into a pipeline
//    stage; one elected thread issues ceil(dim/64)*4 tcgen05.mma (M=256, N=ld_pad, K=16) into one of
//    two TMEM accumulators (128 lanes x 256 fp32 columns each = all 512 TMEM columns), so the epilogue
//    of chunk t overlaps the MMAs of chunk t+1.  A chunk longer than 256 tokens (H = 2) is two
//    N <= 256 halves, one per accumulator, drained by the same epilogue warps (running max carried).
//  * Epilogue: warp w reads TMEM lanes 32*(w%4)..+31 = 32 token rows of one query; each thread (one
//    query token i) reduces max over the chunk's real columns j < len_c (columns >= len_c are never
//    read: reading R2), the warp then sums over real query tokens i < len_q (butterfly shuffle, fixed
//    order: R3; a query of QW warps adds its warps' sums in warp order through shared memory).  The
//    q x d token-similarity tensor never leaves TMEM.
//  * MODE 0 writes S[q][c] (dense scores: ColTrast in-batch matrix a10, test export).
//    MODE 1 keeps a per-(unit, query) top-k in registers (KR x 32 lanes, sortable 64-bit keys
//    (orderable(score) << 32 | ~id): larger key = higher score, then lower id -- reading R6) and writes
//    it to partial[p][grp][q][0..k) at the end of the unit (a6); topk_merge.cuh merges them (a7).
//    MODE 2 is MODE 0 plus the argmax doc token of every max (the N1 backward's forward).
#pragma once
#include <cuda.h>
#include <cuda_bf16.h>
#include <cstdint>

#include "../ptx.cuh"

namespace hiper {

struct MaxsimArgs {
  int32_t n_q;       // real queries
  int32_t n_groups;  // row groups (8 / QW queries each)
  int32_t n_parts;   // P
  int32_t ld_pad;    // token rows per chunk (multiple of 16, <= 512; > 256: two MMA halves)
  int32_t num_kb;    // ceil(dim / 64) (TMA zero-fills the columns past dim)
  int32_t k;         // top-k (MODE 1)
  int32_t n_stages;  // B pipeline stages
  uint32_t a_bytes;  // one A buffer (num_kb * 16 KiB)
  uint32_t stage_bytes;  // box_rows * 128 * num_kb (this CTA's rows of one chunk / chunk half)
  uint32_t box_rows;     // TMA box rows of the corpus map (ld_pad / 2, or 128 for ld_pad > 256)
  int32_t a_bufs;        // A tile buffers (2 = double-buffered across units, 1 for large dims)
  int32_t q_pad;         // padded query count = n_groups * 8 / QW (partial-list row stride)
  int64_t n_chunks;
  int64_t id_base;
  const int32_t* q_lens;  // device [n_q]
  const int32_t* d_lens;  // device [n_chunks]
  float* scores;          // MODE 0: [n_q][score_ld]
  int64_t score_ld;
  uint64_t* partial;      // MODE 1: [P][2][q_pad][k]
  uint32_t* progress;     // pair kernel: [n_pairs] progress words for L2 lockstep, or nullptr
  uint8_t* amax;          // MODE 2: [n_q][score_ld][32] argmax doc-token index of every max
  int32_t window;         // chunks a pair may run ahead of the slowest pair (lockstep window)
  // packed layout (N4, PACKED kernels): slot c of the kernel is tile c of a length-bucketed packed
  // corpus, described by a 128-B record recs[c][0..32): w0 = n_rows | n_ent << 16 (n_rows a multiple
  // of 16, <= 256; n_ent <= 16 chunks), w1 = start mask (bit g: a chunk begins at column group g of
  // 16), w4 = first packed row, w16 + e = chunk index of slot e (slots in column order).  The
  // padding rows of a chunk's last 16-row group repeat its last real row (no column masking).
  const uint32_t* recs;
  unsigned long long* stats;  // HIPER_PIPE_STATS diagnostics (see pooled_sm100_pair.cuh), or nullptr
  int32_t ls_mask;            // L2 lockstep: publish / check every ls_mask + 1 chunks (a power of two)
  int32_t late_release;       // A/B only (HIPER_LATE_RELEASE=1): release the accumulator after the
                              // drain's arithmetic instead of after its last TMEM load
};

// 12 warps: 0-7 epilogue groups 0/1, 8 TMEM allocator, 10 TMA producer, 11 MMA issuer.
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
// Running max and argmax (lowest column on exact ties) with one running pair per thread.  The block
// max is the max of its two 32-column halves (FMNMX3 chains); only a block that raises the running max
// is scanned for its lowest column attaining it: the first half holding the max is selected (32 SEL)
// and scanned downwards with == in 8 interleaved chains (64 instructions instead of 128 for the whole
// block -- the scan is issue-bound, and the warp runs it whenever any lane improves).  The lowest
// match is always a real column: the max is attained by one, and padded columns (index >= rem) come
// after every real one.
__device__ __forceinline__ void max64_arg1(const uint32_t (&v)[64], float& m, int& ix, int base,
                                           int rem) {
  float h[2][2] = {{-INFINITY, -INFINITY}, {-INFINITY, -INFINITY}};
  if (rem >= 64) {
#pragma unroll
    for (int half = 0; half < 2; ++half)
#pragma unroll
      for (int i = 0; i < 32; i += 4)
#pragma unroll
        for (int c = 0; c < 2; ++c)
          h[half][c] = fmaxf(fmaxf(h[half][c], __uint_as_float(v[32 * half + i + 2 * c])),
                             __uint_as_float(v[32 * half + i + 2 * c + 1]));
  } else {
#pragma unroll
    for (int i = 0; i < 64; ++i) {
      const float x = (i < rem) ? __uint_as_float(v[i]) : -INFINITY;
      h[i >> 5][i & 1] = fmaxf(h[i >> 5][i & 1], x);
    }
  }
  const float h0 = fmaxf(h[0][0], h[0][1]), h1 = fmaxf(h[1][0], h[1][1]);
  const float mb = fmaxf(h0, h1);
  if (mb > m) {
    const bool upper = !(h0 == mb);  // ties go to the lower half
    int jc[8];
#pragma unroll
    for (int c = 0; c < 8; ++c) jc[c] = 32;
#pragma unroll
    for (int i = 31; i >= 0; --i) {
      const float x = __uint_as_float(upper ? v[32 + i] : v[i]);
      jc[i & 7] = (x == mb) ? i : jc[i & 7];
    }
    const int j = min(min(min(jc[0], jc[1]), min(jc[2], jc[3])), min(min(jc[4], jc[5]), min(jc[6], jc[7])));
    m = mb;
    ix = base + (upper ? 32 : 0) + j;
  }
}

}  // namespace hiper
