/*
 * hiper.h -- C ABI of the B200-native ColTrast late-interaction (MaxSim) hot path.
 *
 * The method (HiPerRAG, arXiv 2505.04846, /root/reference/PAPER.md):
 *   S(q, d) = sum_{i < len_q} max_{j < len_d} < q_i , d_j >                      (§2.2,
 *   over L2-normalised token embeddings ("cosine per token pair")    PAPER.md:228 Fig.3B,
 *                                                                                  PAPER.md:241 §3.2.1)
 * used (i) for exact top-k retrieval over a chunk index ("semantic search in the vector database to
 * identify the nearest neighbors", §2.3) and (ii) for the in-batch B x B score matrix of
 * the ColTrast late-interaction loss L_LI ("L_LI is maxsim loss", §3.2.1).
 * Readings of every gap (length masking, normalisation recipe, ties, padding) are DESIGN.md R1-R17.
 *
 * Conventions (all entry points):
 *  - Never throws; every call returns hiper_status.  hiper_last_error() gives a thread-local detail
 *    string for the last failing call on this thread.
 *  - "device" pointers are CUDA device memory on the current device; "HOST" pointers are ordinary host
 *    memory (read synchronously during the call, never retained).  Length arrays and pos_idx are small
 *    HOST arrays so validation is eager; all device work is enqueued asynchronously on `stream`.
 *  - Errors detectable on the host are returned before any launch, with outputs untouched.  A CUDA or
 *    NCCL failure returns HIPER_ERR_CUDA / HIPER_ERR_NCCL and leaves outputs undefined.
 *  - Token tensors are row-major [n][max_len][dim] (dim contiguous), float32 or bfloat16.  Rows
 *    j >= len of an item are ignored (never read as zero vectors into a max, reading R2/R3).
 *  - Scores are computed with bf16 operands and fp32 accumulation (tcgen05 tensor cores, sm_100a).
 *  - Supported shapes: token dim % 16 == 0 and <= 256 (pooled: <= 4096); q_max_len <= 128;
 *    chunk max_len <= 512 (HIPER_PACKED: <= 256); 1 <= k <= 128; global ids < 2^32 - 1;
 *    n * roundup(max_len,16) < 2^31 per index.  Anything else returns HIPER_ERR_UNSUPPORTED.
 *    (Narrower: the N1 backward takes q_max_len <= 32, d_max_len <= 256, dim 64 or 128; the N3
 *    rerank takes token dim <= 128, q_max_len <= 32, max_len <= 256.)
 *  - No CPU fallback exists: without an sm_100 device every compute call returns HIPER_ERR_UNSUPPORTED
 *    or HIPER_ERR_CUDA.
 */
#ifndef HIPER_H_
#define HIPER_H_

#include <stddef.h>
#include <stdint.h>

#if defined(HIPER_BUILD)
#define HIPER_API __attribute__((visibility("default")))
#else
#define HIPER_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st* hiper_stream_t; /* == cudaStream_t; NULL = legacy default stream */

typedef enum {
  HIPER_OK = 0,
  HIPER_ERR_INVALID_ARG = 1,     /* null pointer, k < 1, n < 0, bad flags, ... */
  HIPER_ERR_DIM_MISMATCH = 2,    /* SPEC DimensionMismatch: query dim != index dim */
  HIPER_ERR_EMPTY_TOKENS = 3,    /* SPEC EmptyTokenList: some len == 0 */
  HIPER_ERR_EMPTY_BATCH = 4,     /* SPEC EmptyBatch: n_q == 0 for the loss */
  HIPER_ERR_BAD_TEMPERATURE = 5, /* SPEC NonPositiveTemperature: tau <= 0 or not finite */
  HIPER_ERR_BAD_POSITIVE = 6,    /* SPEC InvalidPositiveIndex */
  HIPER_ERR_NONFINITE = 7,       /* SPEC "all entries finite" */
  HIPER_ERR_ZERO_VECTOR = 8,     /* SPEC ZeroVector: a real row of norm 0 under NORM */
  HIPER_ERR_OUT_OF_MEMORY = 9,
  HIPER_ERR_CUDA = 10,
  HIPER_ERR_NCCL = 11,
  HIPER_ERR_UNSUPPORTED = 12,    /* shape/device outside the supported set above */
  HIPER_ERR_WORKSPACE = 13       /* workspace NULL / too small / misaligned (needs 1024-B alignment) */
} hiper_status;

typedef enum { HIPER_F32 = 0, HIPER_BF16 = 1 } hiper_dtype;

enum {
  /* Rows are already unit-norm: skip NORM, store RNE_bf16(x) (reading R12). */
  HIPER_ASSUME_NORMALIZED = 1u,
  /* Reject non-finite entries (always on for hiper_index_build; opt-in for queries). */
  HIPER_CHECK_FINITE = 2u,
  /* hiper_index_build only: zero-copy.  The index references the caller's bf16 token buffer, which must
   * have max_len % 16 == 0, 16-byte alignment, outlive the index and not be modified.  NORM (unless
   * ASSUME_NORMALIZED) is applied IN PLACE and rows j >= len are zeroed in place. */
  HIPER_BORROW_TOKENS = 4u,
  /* Query-side calls: synchronise `stream` after query preparation and return HIPER_ERR_ZERO_VECTOR /
   * HIPER_ERR_NONFINITE if a real query row is zero / non-finite.  Without it the same condition is
   * recorded in the workspace status word (hiper_workspace_status) and scores are undefined. */
  HIPER_VALIDATE_SYNC = 8u,
  /* hiper_index_build only (NEXT N4, variable-length chunks from semantic chunking):
   * length-bucketed packed layout.  Chunk c occupies roundup(lens[c], 16) rows of a tile of <= 256
   * rows (hiper_pack_plan); the MaxSim kernel's MMA N is the tile's row count, so padded token
   * columns are neither stored nor multiplied.  The rows past a chunk's length inside its 16-row slot
   * are written as copies of its last real row, so the kernel needs no column masking (a repeated
   * column cannot change a maximum).  Results are those of the dense layout, also as the token
   * index of hiper_two_stage_topk (which reads chunks by id through a per-chunk row table the
   * index keeps, 8 B per chunk).  With HIPER_BORROW_TOKENS as well, `tokens` is the caller's bf16 buffer
   * ALREADY in the packed layout ([n_rows][dim], chunk c's token j at row row0(tile) + col + j as
   * hiper_pack_plan(lens) places it; rows past a chunk's length inside its 16-row slot are ignored
   * and overwritten as above), NORM'd in place: no second copy of the corpus (the paper-scale 16.4M-chunk corpus,
   * PAPER.md:564, at 110 GB per GPU on 4 GPUs).  The buffer must hold n_rows rows and outlive the
   * index. */
  HIPER_PACKED = 16u,
  /* hiper_index_build only: a POOLED index (the a12 limit case; "cosine similarity on
   * the pooled embeddings"): one vector per item (max_len must be 1), scored by the pooled GEMM kernel,
   * queried with q_max_len 1.  dim % 16 == 0, <= 4096.  Without this flag a max_len-1 index is a token
   * index like any other (any query length scores against its single row). */
  HIPER_POOLED = 32u
};

typedef struct hiper_index_s hiper_index; /* opaque; immutable after build; shareable by readers */
typedef struct hiper_comm_s hiper_comm;   /* opaque; owns one ncclComm_t */

HIPER_API const char* hiper_status_string(hiper_status s);
HIPER_API const char* hiper_last_error(void);
HIPER_API int32_t hiper_version(void); /* major*10000 + minor*100 + patch */

/* ------------------------------------------------------------------ multi-GPU (corpus sharding)
 * One process per GPU.  Rank 0 calls hiper_comm_unique_id and broadcasts the 128 bytes (the Python
 * binding uses torch.distributed); every rank then calls hiper_comm_create.  The communicator carries
 * exactly one collective per query batch: an ncclAllGather of each shard's local top-k keys
 * (BASELINE.json north_star: "merged with one NCCL all-gather over NVLink"). */
/* The corpus shard plan (pure host function): rank r of `world` holds chunks [c0, c1) =
 * [r * n / world, (r + 1) * n / world) -- contiguous, sizes within one of each other; builds its index
 * with id_base = c0. */
HIPER_API hiper_status hiper_shard_range(int64_t n, int32_t world, int32_t rank, int64_t* c0, int64_t* c1);
HIPER_API hiper_status hiper_comm_unique_id(uint8_t id[128]);
HIPER_API hiper_status hiper_comm_create(const uint8_t id[128], int32_t world, int32_t rank, int32_t device,
                               hiper_comm** out);
HIPER_API hiper_status hiper_comm_destroy(hiper_comm* comm);
HIPER_API hiper_status hiper_comm_info(const hiper_comm* comm, int32_t* world, int32_t* rank);

/* ------------------------------------------------------------------ step a1: corpus layout
 * hiper_index_build: lay out a chunk corpus for scoring ("chunk embeddings are stored in a vector
 * database ... each linked to a unique ID"; SPEC.md:184-192 build_index).
 *   tokens  device [n][max_len][dim] (dtype), finite.
 *   lens    HOST [n], 1 <= lens[c] <= max_len (EmptyTokenList otherwise).
 *   id_base global id of chunk 0 of this shard; chunk c gets id id_base + c.
 * Result layout (owned by the index unless BORROW): bf16 [n][ld_pad][dim], ld_pad = roundup(max_len,16),
 * row j < lens[c] = NORM(tokens[c][j]) (R1), rows j >= lens[c] = 0; lens kept on device.
 * Synchronises `stream` once at the end (build-time validation of NONFINITE / ZERO_VECTOR).
 * n == 0 gives a valid empty index (searches return all padding). */
HIPER_API hiper_status hiper_index_build(const void* tokens, hiper_dtype dtype, const int32_t* lens, int64_t n,
                               int32_t max_len, int32_t dim, int64_t id_base, uint32_t flags,
                               hiper_stream_t stream, hiper_index** out);
HIPER_API hiper_status hiper_index_destroy(hiper_index* idx);
/* Any output pointer may be NULL.  layout: device bf16 [n][ld_pad][dim]; lens_dev: device int32 [n]. */
HIPER_API hiper_status hiper_index_info(const hiper_index* idx, int64_t* n, int32_t* max_len, int32_t* dim,
                              int32_t* ld_pad, int64_t* id_base, const void** layout,
                              const int32_t** lens_dev);

/* NEXT N4: the packing plan HIPER_PACKED uses (pure host function; no device needed).
 *   lens       HOST [n], 1..256.
 *   tiles_out  HOST int32 [n][4] capacity: tile t = {row0, n_rows, e0, e1}, n_rows % 16 == 0,
 *              n_rows <= 256, tiles contiguous (row0 of t+1 = row0 + n_rows of t).
 *   ents_out   HOST int32 [n][2]: entry e = {chunk index, (col << 16) | len}: the chunk's token j is
 *              packed row row0 + col + j of its tile; entries [e0, e1) of a tile are its chunks,
 *              every chunk appears in exactly one entry, col % 16 == 0.
 *   n_tiles, n_rows: counts (either may be NULL).
 * Greedy largest-first fill over 16 width buckets; deterministic in lens. */
HIPER_API hiper_status hiper_pack_plan(const int32_t* lens, int64_t n, int32_t* tiles_out, int32_t* ents_out,
                             int64_t* n_tiles, int64_t* n_rows);
/* Packing of a built index (test support; any output may be NULL).  packed = 0 for a dense index.
 * layout (hiper_index_info) is then bf16 [n_rows][dim]; tiles_dev int32 [n_tiles][4] and ents_dev
 * int32 [n][2] are device copies of the hiper_pack_plan tables. */
HIPER_API hiper_status hiper_index_pack_info(const hiper_index* idx, int32_t* packed, int64_t* n_tiles,
                                   int64_t* n_rows, const void** tiles_dev, const void** ents_dev);

/* ------------------------------------------------------------------ step a2: query preparation
 * NORM every real query row into the kernel's query layout: out device bf16 [n_q_pad][QS][dim] with
 * QS = 32 / 64 / 128 for q_max_len <= 32 / 64 / 128 (one, two or four warps of TMEM lanes per query)
 * and n_q_pad = roundup(n_q, 256 / QS); rows i >= q_lens[q] and queries q >= n_q are zero.  status: device
 * uint32 (bit 0: zero row, bit 1: non-finite row), OR-ed, may be NULL.  Exposed so the layout can be
 * checked bitwise against the oracle's NORM; the search/loss entry points call it internally. */
HIPER_API hiper_status hiper_prepare_queries(const void* q_tokens, hiper_dtype dtype, const int32_t* q_lens,
                                   int32_t n_q, int32_t q_max_len, int32_t dim, uint32_t flags,
                                   void* out_layout, uint32_t* status, hiper_stream_t stream);

/* ------------------------------------------------------------------ steps a2-a9: exact top-k
 * hiper_maxsim_topk: for every query, the k chunks of highest S(q, c) over this shard (comm == NULL)
 * or over all shards of `comm` (every rank passes the same queries and receives the identical global
 * result).  Ordering: score descending, then global id ascending (R6).  When
 * k > number of chunks the tail is (score -inf, id -1) (R7).
 *   q_tokens device [n_q][q_max_len][dim]; q_lens HOST [n_q] in 1..q_max_len.
 *   workspace device, >= hiper_maxsim_topk_workspace_size(idx, n_q, k, comm) bytes, 1024-B aligned,
 *             caller-owned (e.g. torch allocator), not used concurrently by another call.
 *   out_scores device float [n_q][k]; out_ids device int64 [n_q][k].
 * Launches: query prep, the fused TMA/tcgen05 MaxSim + per-CTA top-k kernel, the top-k merge kernel
 * (+ ncclAllGather and a second merge when comm != NULL). */
HIPER_API size_t hiper_maxsim_topk_workspace_size(const hiper_index* idx, int32_t n_q, int32_t k,
                                        const hiper_comm* comm);
HIPER_API hiper_status hiper_maxsim_topk(const hiper_index* idx, const void* q_tokens, hiper_dtype dtype,
                               const int32_t* q_lens, int32_t n_q, int32_t q_max_len, int32_t dim,
                               int32_t k, uint32_t flags, const hiper_comm* comm, void* workspace,
                               size_t workspace_bytes, float* out_scores, int64_t* out_ids,
                               hiper_stream_t stream);

/* ------------------------------------------------------------------ step a8, in two halves
 * The cross-GPU merge of hiper_maxsim_topk(comm != NULL) is: every rank's local top-k as sortable
 * 64-bit keys -> one ncclAllGather into [world][n_q][k] -> the same merge + decode on every rank.  The
 * two halves are exported so the merge can be driven (and tested against the oracle) without NCCL:
 * nearest neighbours over the whole store (§2.3) from per-shard lists (north star:
 * "merged with one NCCL all-gather").
 * Key format: (orderable(score) << 32) | (~(uint32)global_id), orderable(f) = bits(f) ^ (f < 0 ?
 * 0xFFFFFFFF : 0x80000000); a larger key = a higher score, then a lower id (R6); key 0 = empty slot.
 *
 * hiper_maxsim_topk_keys: as hiper_maxsim_topk with comm == NULL, but writes this shard's top-k as keys,
 *   out_keys device uint64 [n_q][k] (descending; 0-padded when k > n).  Workspace: as
 *   hiper_maxsim_topk_workspace_size(idx, n_q, k, NULL).
 * hiper_topk_merge_keys: lists device uint64 [n_lists][n_q][k] (each [n_q][k] block sorted descending,
 *   as written by hiper_maxsim_topk_keys or gathered by ncclAllGather) -> the top-k of their union,
 *   decoded: out_scores device float [n_q][k], out_ids device int64 [n_q][k] (padding -inf / -1).
 *   1 <= k <= 128; n_lists >= 0 (0 gives all padding).  Bitwise independent of the list order. */
HIPER_API hiper_status hiper_maxsim_topk_keys(const hiper_index* idx, const void* q_tokens,
                                    hiper_dtype dtype, const int32_t* q_lens, int32_t n_q,
                                    int32_t q_max_len, int32_t dim, int32_t k, uint32_t flags,
                                    void* workspace, size_t workspace_bytes, uint64_t* out_keys,
                                    hiper_stream_t stream);
HIPER_API hiper_status hiper_topk_merge_keys(const uint64_t* lists, int32_t n_lists, int32_t n_q,
                                   int32_t k, float* out_scores, int64_t* out_ids,
                                   hiper_stream_t stream);

/* ------------------------------------------------------------------ dense scores (test support + a10)
 * out_scores device float [n_q][n] = S(q, c) for every query and every chunk of the index. */
HIPER_API size_t hiper_maxsim_scores_workspace_size(const hiper_index* idx, int32_t n_q);
HIPER_API hiper_status hiper_maxsim_scores(const hiper_index* idx, const void* q_tokens, hiper_dtype dtype,
                                 const int32_t* q_lens, int32_t n_q, int32_t q_max_len, int32_t dim,
                                 uint32_t flags, void* workspace, size_t workspace_bytes,
                                 float* out_scores, hiper_stream_t stream);

/* ------------------------------------------------------------------ steps a10-a11: ColTrast L_LI
 * In-batch MaxSim scores S[i][j] = S(Q_i, D_j) (i < n_q, j < n_d) and the InfoNCE loss over them
 * ("We apply LI loss to the local rank only"; SPEC.md:339-347 li_loss):
 *   z_ij = S_ij / temperature;  l_i = logsumexp_j z_ij - z_{i,pos_i};  L = (1/n_q) sum_i l_i
 * computed in fp32 with a max shift and the log1p form of DESIGN.md R13; fixed-order (deterministic)
 * reductions.  temperature == 1 reproduces SPEC li_loss exactly (R9).
 *   q_tokens device [n_q][q_max_len][dim], d_tokens device [n_d][d_max_len][dim] (same dtype);
 *   q_lens / d_lens HOST; pos_idx HOST [n_q] or NULL (= diagonal, needs n_d >= n_q).
 *   out_scores device float [n_q][n_d] or NULL; out_loss device float scalar (not NULL).
 *   workspace >= hiper_coltrast_workspace_size(...) bytes, 1024-B aligned. */
HIPER_API size_t hiper_coltrast_workspace_size(int32_t n_q, int32_t n_d, int32_t d_max_len, int32_t dim);
HIPER_API hiper_status hiper_coltrast_scores_loss(const void* q_tokens, const int32_t* q_lens, int32_t n_q,
                                        int32_t q_max_len, const void* d_tokens,
                                        const int32_t* d_lens, int32_t n_d, int32_t d_max_len,
                                        int32_t dim, hiper_dtype dtype, uint32_t flags,
                                        const int32_t* pos_idx, float temperature,
                                        void* workspace, size_t workspace_bytes,
                                        float* out_scores, float* out_loss, hiper_stream_t stream);

/* ------------------------------------------------------------------ NEXT N2: the full ColTrast loss
 * L = (L_LI + L_C) / 2 ("The total loss per iteration is L = (L_LI + L_C)/2").
 *  L_LI: as hiper_coltrast_scores_loss over the local rank's b queries vs its b positives (token level,
 *        diagonal positives, temperature tau_li; "We apply LI loss to the local rank only").
 *  L_C:  InfoNCE over cos(pooled q_i, c_j) / tau_c (SimCSE form).  The candidates c_j
 *        are the pooled positives of ALL ranks of `comm`, gathered with one ncclAllGather ("pooled
 *        embeddings from all ranks are gathered, and loss is calculated with the local rank compared
 *        to min(N, W) samples"): the local b positives first, then the other ranks in
 *        (rank, position) order, truncated to m = min(n_max, W), W = world * b.
 *        Query i's positive is candidate i.
 *   q_tokens/d_tokens device [b][q_max_len|d_max_len][dim]; q_lens/d_lens HOST [b];
 *   q_pooled/d_pooled device [b][dp] (any scale: NORM'd inside), dp % 64 == 0;
 *   n_max >= b (else HIPER_ERR_INVALID_ARG, SPEC NTooSmall); comm may be NULL (W = b).
 *   out_losses device float[3] = {L_LI, L_C, L}; out_scores_c device float [b][m] or NULL;
 *   out_m HOST int32 (may be NULL) receives m.  Every rank of comm must call it (collective). */
HIPER_API size_t hiper_coltrast_loss_workspace_size(int32_t b, int32_t d_max_len, int32_t dim,
                                                    int32_t dp, int32_t n_max,
                                                    const hiper_comm* comm);
HIPER_API hiper_status hiper_coltrast_loss(const void* q_tokens, const int32_t* q_lens,
                                           int32_t q_max_len, const void* d_tokens,
                                           const int32_t* d_lens, int32_t d_max_len, int32_t dim,
                                           const void* q_pooled, const void* d_pooled, int32_t dp,
                                           int32_t b, hiper_dtype dtype, uint32_t flags,
                                           int32_t n_max, float tau_li, float tau_c,
                                           const hiper_comm* comm, void* workspace,
                                           size_t workspace_bytes, float* out_losses,
                                           float* out_scores_c, int32_t* out_m,
                                           hiper_stream_t stream);

/* The gather of L_C's candidates: with a communicator of ranks on one node, every rank NORMs its
 * pooled passages straight into its own window -- device memory exported once with CUDA IPC and mapped
 * by every peer when the communicator is first used here (collective) -- and publishes a ready epoch;
 * one kernel then reads the local and the peers' windows over NVLink in min(N, W) order into the
 * candidate matrix (no ncclAllGather, no reorder copies).  Without IPC (ranks on different nodes), or
 * with HIPER_N2_NCCL set, an ncclAllGather feeds the same kernel.
 *
 * hiper_coltrast_loss_simulated (test support): the same computation for rank `rank` of `world`
 * simulated ranks on ONE GPU: d_pooled_all is device [world][b][dp], every simulated rank's passages
 * (each rank's own are its slice); everything else as hiper_coltrast_loss. */
HIPER_API size_t hiper_coltrast_loss_simulated_workspace_size(int32_t b, int32_t d_max_len, int32_t dim,
                                                              int32_t dp, int32_t n_max, int32_t world);
HIPER_API hiper_status hiper_coltrast_loss_simulated(
    const void* q_tokens, const int32_t* q_lens, int32_t q_max_len, const void* d_tokens,
    const int32_t* d_lens, int32_t d_max_len, int32_t dim, const void* q_pooled,
    const void* d_pooled_all, int32_t dp, int32_t b, hiper_dtype dtype, uint32_t flags,
    int32_t n_max, float tau_li, float tau_c, int32_t world, int32_t rank, void* workspace,
    size_t workspace_bytes, float* out_losses, float* out_scores_c, int32_t* out_m,
    hiper_stream_t stream);

/* ------------------------------------------------------------------ NEXT N1: backward of L_LI
 * Forward exactly as hiper_coltrast_scores_loss (the fused kernel additionally records the argmax
 * doc token of every max), then the gradient of L_LI with respect to the RAW token inputs:
 *   G_ij = (softmax_j(S_i/tau)_j - [j == pos_i]) / (n_q tau);  a(i,t,j) = argmax_u <qn_it, dn_ju>
 *   (lowest u on exact ties);  g_q(i,t) = sum_j G_ij dn_{j,a};  g_d(j,u) = sum_{i,t: a=u} G_ij qn_it;
 *   grad_x = (g - y (y.g)) / ||x||, y = x/||x||  (NORM's Jacobian; identity with ASSUME_NORMALIZED).
 * (Training the ColTrast objective by backpropagation.)
 *   grad_q device float [n_q][q_max_len][dim], grad_d device float [n_d][d_max_len][dim]; padding
 *   rows are 0.  Requires the CTA-pair kernel (the default).  dim in {64, 128}. */
HIPER_API size_t hiper_coltrast_grad_workspace_size(int32_t n_q, int32_t n_d, int32_t d_max_len,
                                                    int32_t dim);
HIPER_API hiper_status hiper_coltrast_scores_loss_grad(
    const void* q_tokens, const int32_t* q_lens, int32_t n_q, int32_t q_max_len,
    const void* d_tokens, const int32_t* d_lens, int32_t n_d, int32_t d_max_len, int32_t dim,
    hiper_dtype dtype, uint32_t flags, const int32_t* pos_idx, float temperature, void* workspace,
    size_t workspace_bytes, float* out_scores, float* out_loss, float* grad_q, float* grad_d,
    hiper_stream_t stream);

/* ------------------------------------------------------------------ NEXT N3: two-stage retrieval
 * Stage 1: pooled-cosine top-k1 over pooled_idx (built with max_len 1: the paper's deployed
 * retrieval); stage 2: exact MaxSim re-scoring of those k1 candidates over
 * token_idx, the token rows of the SAME chunks (same n and id_base; dense or HIPER_PACKED), keeping
 * the final top-k
 * (ColBERTv2's retrieve-then-rerank; SPEC.md:268-276 rerank; score desc, id asc).
 *   q_pooled device [n_q][pooled dim]; q_tokens device [n_q][q_max_len][token dim]; q_lens HOST.
 *   1 <= k <= k1 <= 128.  Stage 2 computes each query's own k1 candidates exactly once (a gather of
 *   their token rows, HBM-bound); token dim <= 128, q_max_len <= 32, max_len <= 256.
 *   comm: NULL = this shard only.  With a communicator every rank passes the same queries and its
 *   own shard (both indexes with the shard's id_base): stage 1 is the global pooled top-k1 (one
 *   all-gather), each rank re-scores the candidates it owns, and one more all-gather + merge gives
 *   every rank the identical global top-k -- bitwise the single-GPU result on the whole corpus. */
HIPER_API size_t hiper_two_stage_workspace_size(const hiper_index* pooled_idx,
                                                const hiper_index* token_idx, int32_t n_q,
                                                int32_t k1, const hiper_comm* comm);
HIPER_API hiper_status hiper_two_stage_topk(const hiper_index* pooled_idx,
                                            const hiper_index* token_idx, const void* q_pooled,
                                            const void* q_tokens, hiper_dtype dtype,
                                            const int32_t* q_lens, int32_t n_q, int32_t q_max_len,
                                            int32_t k1, int32_t k, uint32_t flags,
                                            const hiper_comm* comm, void* workspace,
                                            size_t workspace_bytes, float* out_scores,
                                            int64_t* out_ids, hiper_stream_t stream);

/* Loss kernel alone over a given device score matrix S [n_q][n_d] (test support: isolates a11). */
HIPER_API hiper_status hiper_infonce_loss(const float* scores, int32_t n_q, int32_t n_d,
                                const int32_t* pos_idx, float temperature, void* workspace,
                                size_t workspace_bytes, float* out_loss, hiper_stream_t stream);

/* Synchronise `stream` and report the device-side status word of a query-side workspace:
 * HIPER_OK, HIPER_ERR_ZERO_VECTOR or HIPER_ERR_NONFINITE. */
HIPER_API hiper_status hiper_workspace_status(const void* workspace, hiper_stream_t stream);

/* Number of kernels the last successful compute call on this thread enqueued (bench evidence). */
HIPER_API int32_t hiper_last_launch_count(void);

/* Live per-kernel timing for the roofline report: while enabled, every launch of the fused MaxSim
 * kernel is bracketed by CUDA events on its own stream.  hiper_profile_read synchronises on the
 * recorded events, returns the summed kernel milliseconds and the number of launches since the last
 * read, and resets the record. */
HIPER_API void hiper_profile_enable(int32_t on);
HIPER_API hiper_status hiper_profile_read(double* maxsim_ms, int32_t* n_launches);
/* The same for one kernel class only (the others stay recorded): HIPER_PROF_MAXSIM (the fused MaxSim
 * kernel), HIPER_PROF_POOLED (the pooled GEMM + top-k kernel), HIPER_PROF_RERANK (the N3 gather). */
enum { HIPER_PROF_MAXSIM = 0, HIPER_PROF_POOLED = 1, HIPER_PROF_RERANK = 2 };
HIPER_API hiper_status hiper_profile_read_tagged(int32_t tag, double* ms, int32_t* n_launches);

#ifdef __cplusplus
}
#endif
#endif /* HIPER_H_ */
