// hiper_api.cu -- host side of the C ABI declared in include/hiper.h.
//
// Validation (eager, on host arrays), workspace carving, TMA tensor-map encoding, launches and the
// NCCL all-gather.  No computation of the method happens on the host: every step runs in the kernels
// under kernels/.  There is no CPU fallback: without an sm_100 device every compute entry point fails.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <nccl.h>
#include <nvtx3/nvToolsExt.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <numeric>
#include <string>
#include <type_traits>
#include <utility>
#include <vector>

#include "../../include/hiper.h"
#include "kernels/infonce.cuh"
#include "kernels/maxsim_backward.cuh"
#include "kernels/maxsim_sm100_pair.cuh"
#include "kernels/pooled_sm100_pair.cuh"
#include "kernels/pooled_cs_sm100.cuh"
#include "kernels/rerank_gather.cuh"
#include "kernels/peer_gather.cuh"
#include "kernels/norm_layout.cuh"
#include "kernels/topk_merge.cuh"

using namespace hiper;

// ============================================================================ errors
static thread_local std::string g_last_error;
static thread_local int32_t g_launches = 0;

static hiper_status fail(hiper_status s, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_last_error = buf;
  return s;
}

#define CUDA_TRY(expr)                                                                        \
  do {                                                                                        \
    cudaError_t _e = (expr);                                                                  \
    if (_e != cudaSuccess)                                                                    \
      return fail(_e == cudaErrorMemoryAllocation ? HIPER_ERR_OUT_OF_MEMORY : HIPER_ERR_CUDA, \
                  "%s: %s (%s:%d)", #expr, cudaGetErrorString(_e), __FILE__, __LINE__);       \
  } while (0)

#define TRY(expr)                        \
  do {                                   \
    hiper_status _s = (expr);            \
    if (_s != HIPER_OK) return _s;       \
  } while (0)

extern "C" const char* hiper_status_string(hiper_status s) {
  switch (s) {
    case HIPER_OK: return "HIPER_OK";
    case HIPER_ERR_INVALID_ARG: return "HIPER_ERR_INVALID_ARG";
    case HIPER_ERR_DIM_MISMATCH: return "HIPER_ERR_DIM_MISMATCH";
    case HIPER_ERR_EMPTY_TOKENS: return "HIPER_ERR_EMPTY_TOKENS";
    case HIPER_ERR_EMPTY_BATCH: return "HIPER_ERR_EMPTY_BATCH";
    case HIPER_ERR_BAD_TEMPERATURE: return "HIPER_ERR_BAD_TEMPERATURE";
    case HIPER_ERR_BAD_POSITIVE: return "HIPER_ERR_BAD_POSITIVE";
    case HIPER_ERR_NONFINITE: return "HIPER_ERR_NONFINITE";
    case HIPER_ERR_ZERO_VECTOR: return "HIPER_ERR_ZERO_VECTOR";
    case HIPER_ERR_OUT_OF_MEMORY: return "HIPER_ERR_OUT_OF_MEMORY";
    case HIPER_ERR_CUDA: return "HIPER_ERR_CUDA";
    case HIPER_ERR_NCCL: return "HIPER_ERR_NCCL";
    case HIPER_ERR_UNSUPPORTED: return "HIPER_ERR_UNSUPPORTED";
    case HIPER_ERR_WORKSPACE: return "HIPER_ERR_WORKSPACE";
  }
  return "HIPER_ERR_UNKNOWN";
}
// NVTX range around every ABI entry point (header-only NVTX3: a no-op unless a profiler such as
// nsys / ncu --nvtx is attached), so a timeline shows which library call each kernel belongs to.
struct HiperRange {
  explicit HiperRange(const char* name) { nvtxRangePushA(name); }
  ~HiperRange() { nvtxRangePop(); }
  HiperRange(const HiperRange&) = delete;
  HiperRange& operator=(const HiperRange&) = delete;
};

static constexpr int32_t kMaxK = 128;         // top-k capacity of every list (register / warp lists)
static constexpr int32_t kMaxChunkLen = 512;  // chunk tokens (> 256: two MMA halves per chunk)
static constexpr int32_t kMaxQueryLen = 128;  // query tokens (query slots of 32, 64 or 128 rows)

extern "C" const char* hiper_last_error(void) { return g_last_error.c_str(); }
extern "C" int32_t hiper_version(void) { return 100; }
extern "C" int32_t hiper_last_launch_count(void) { return g_launches; }

// ============================================================================ device helpers
struct DevInfo {
  int device = -1;
  int num_sms = 0;
  int max_smem = 0;
};

static hiper_status device_info(DevInfo& di) {
  int dev = 0;
  CUDA_TRY(cudaGetDevice(&dev));
  int major = 0, minor = 0;
  CUDA_TRY(cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev));
  CUDA_TRY(cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, dev));
  if (major != 10 || minor != 0)
    return fail(HIPER_ERR_UNSUPPORTED, "device %d is sm_%d%d; this build targets sm_100a only", dev,
                major, minor);
  di.device = dev;
  CUDA_TRY(cudaDeviceGetAttribute(&di.num_sms, cudaDevAttrMultiProcessorCount, dev));
  CUDA_TRY(cudaDeviceGetAttribute(&di.max_smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
  return HIPER_OK;
}

typedef CUresult (*PFN_encodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                    const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                    const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                    CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static hiper_status get_encode_fn(PFN_encodeTiled* fn) {
  static PFN_encodeTiled cached = nullptr;
  static std::once_flag once;
  static cudaError_t err = cudaSuccess;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    err = cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
    if (err == cudaSuccess && q == cudaDriverEntryPointSuccess) cached = (PFN_encodeTiled)p;
  });
  if (!cached) return fail(HIPER_ERR_CUDA, "cuTensorMapEncodeTiled unavailable (%s)", cudaGetErrorString(err));
  *fn = cached;
  return HIPER_OK;
}

// 2-D bf16 tensor map over rows of `dim` elements, box = 64 elements x box_rows rows, 128B swizzle.
// box_cols = 64 (128-B rows, SWIZZLE_128B) or 32 (64-B rows, SWIZZLE_64B: the chunk-stationary
// pooled kernel's query stages)
static hiper_status make_tmap(CUtensorMap* map, const void* base, int64_t rows, int32_t dim,
                              int32_t box_rows, int32_t box_cols = 64) {
  PFN_encodeTiled enc;
  TRY(get_encode_fn(&enc));
  cuuint64_t gdim[2] = {(cuuint64_t)dim, (cuuint64_t)rows};
  cuuint64_t gstride[1] = {(cuuint64_t)dim * 2};
  cuuint32_t box[2] = {(cuuint32_t)box_cols, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1u, 1u};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), gdim, gstride,
                   box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   box_cols == 32 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    return fail(HIPER_ERR_CUDA, "cuTensorMapEncodeTiled failed (%d) rows=%lld dim=%d box_rows=%d",
                (int)r, (long long)rows, dim, box_rows);
  return HIPER_OK;
}

// ---------------------------------------------------------------------------- pinned staging ring
// Small HOST arrays (lengths, positives) go to the device through pinned slots so the copy is truly
// asynchronous; a slot is reused only after the event of its previous copy completed.
namespace {
struct StageSlot {
  void* pinned = nullptr;
  size_t cap = 0;
  cudaEvent_t ev = nullptr;
  bool used = false;
};
struct StageRing {
  std::mutex mu;
  StageSlot slot[16];
  int next = 0;
};
StageRing g_rings[64];
}  // namespace

static hiper_status stage_h2d(void* dst, const void* src, size_t bytes, cudaStream_t stream) {
  if (bytes == 0) return HIPER_OK;
  int dev = 0;
  CUDA_TRY(cudaGetDevice(&dev));
  StageRing& ring = g_rings[dev & 63];
  std::lock_guard<std::mutex> lock(ring.mu);
  StageSlot& s = ring.slot[ring.next];
  ring.next = (ring.next + 1) % 16;
  if (s.ev == nullptr) CUDA_TRY(cudaEventCreateWithFlags(&s.ev, cudaEventDisableTiming));
  if (s.used) CUDA_TRY(cudaEventSynchronize(s.ev));
  if (s.cap < bytes) {
    if (s.pinned) CUDA_TRY(cudaFreeHost(s.pinned));
    s.pinned = nullptr;
    size_t cap = std::max<size_t>(bytes, 65536);
    CUDA_TRY(cudaHostAlloc(&s.pinned, cap, cudaHostAllocDefault));
    s.cap = cap;
  }
  memcpy(s.pinned, src, bytes);
  CUDA_TRY(cudaMemcpyAsync(dst, s.pinned, bytes, cudaMemcpyHostToDevice, stream));
  CUDA_TRY(cudaEventRecord(s.ev, stream));
  s.used = true;
  return HIPER_OK;
}

static bool is_device_ptr(const void* p) {
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

static inline size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) once per (device, kernel, size): it is a
// synchronous driver call that otherwise costs microseconds on every launch of a short step.
static cudaError_t set_max_smem(const void* fn, int bytes) {
  static std::mutex mu;
  static std::vector<std::pair<std::pair<int, const void*>, int>> done;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  std::lock_guard<std::mutex> lock(mu);
  for (auto& d : done)
    if (d.first.first == dev && d.first.second == fn && d.second >= bytes) return cudaSuccess;
  e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e == cudaSuccess) done.push_back({{dev, fn}, bytes});
  return e;
}
static inline int64_t round_up(int64_t x, int64_t a) { return (x + a - 1) / a * a; }


// ============================================================================ the index
struct hiper_index_s {
  int64_t n = 0;
  int32_t max_len = 0, ld_pad = 0, dim = 0;
  int64_t id_base = 0;
  int device = -1;
  __nv_bfloat16* tok = nullptr;  // [n][ld_pad][dim]
  bool owns_tok = false;
  int32_t* lens = nullptr;  // device [n]
  bool pooled = false;                // HIPER_POOLED: one vector per item (a12)
  alignas(64) CUtensorMap tmap;       // pooled: box = 64 dims x 128 rows
  alignas(64) CUtensorMap tmap_half;  // tokens: box = 64 dims x (ld_pad/2 | 128) rows (CTA pair)
  // packed layout (HIPER_PACKED, N4): tok is bf16 [n_rows][dim]; tiles/ents as in MaxsimArgs
  bool packed = false;
  int64_t n_tiles = 0, n_rows = 0;
  int4* tiles = nullptr;     // device [n_tiles]: the plan's tiles (hiper_pack_plan layout)
  uint32_t* recs = nullptr;  // device [n_tiles][32]: kernel tile records (tile_records)
  int2* ents = nullptr;   // device [n]
  int64_t* row_of = nullptr;  // device [n]: first packed row of chunk c (two-stage rerank by id)
};

// ---------------------------------------------------------------------------- N4 packing plan
// Chunk c occupies w_c = roundup(len_c, 16) packed rows.  Tiles hold up to kTileRows rows (the MMA N
// of the CTA pair).  Greedy largest-first fill with 16 width buckets: a tile is seeded with a chunk of
// the largest remaining width, then repeatedly takes a chunk of the largest width that still fits.
// Within a bucket chunks go in ascending index order, so the plan is a pure function of lens.
static constexpr int32_t kTileRows = 256;
static hiper_status pack_plan(const int32_t* lens, int64_t n, std::vector<int4>& tiles,
                              std::vector<int2>& ents, std::vector<int64_t>& dst_row, int64_t& rows) {
  constexpr int NB = kTileRows / 16;
  std::vector<std::vector<int32_t>> bucket(NB);
  for (int64_t c = 0; c < n; ++c) {
    if (lens[c] < 1 || lens[c] > kTileRows)
      return fail(HIPER_ERR_INVALID_ARG, "chunk %lld length %d outside 1..%d", (long long)c, lens[c], kTileRows);
    bucket[(lens[c] + 15) / 16 - 1].push_back((int32_t)c);
  }
  std::vector<size_t> head(NB, 0);
  tiles.clear();
  ents.clear();
  ents.reserve((size_t)n);
  dst_row.assign((size_t)n, 0);
  rows = 0;
  int64_t left = n;
  while (left > 0) {
    const int32_t e0 = (int32_t)ents.size();
    int32_t used = 0;
    while (true) {
      int b = std::min(NB, (kTileRows - used) / 16) - 1;
      while (b >= 0 && head[b] == bucket[b].size()) --b;
      if (b < 0) break;
      const int32_t c = bucket[b][head[b]++];
      ents.push_back(make_int2(c, (used << 16) | lens[c]));
      dst_row[c] = rows + used;
      used += 16 * (b + 1);
      --left;
    }
    if (rows + used >= 0x7FFFFFFFll) return fail(HIPER_ERR_UNSUPPORTED, "packed rows >= 2^31; shard the corpus");
    tiles.push_back(make_int4((int32_t)rows, used, e0, (int32_t)ents.size()));
    rows += used;
  }
  return HIPER_OK;
}

// Kernel-side tile records (not part of hiper_pack_plan's ABI): one 128-B record per tile, so the
// kernel reads everything it needs about a tile with ONE coalesced warp load (lane i <- word i):
//   w0 = n_rows | n_ent << 16, w1 = start mask (bit g: a chunk begins at column group g; also set
//   for every group past n_rows, so no chunk's suffix max reaches them), w4 = row0,
//   w16 + e = chunk of slot e.  (No per-group valid-column counts: the padding rows of a chunk's
//   last group repeat its last real row, pack_pad_replicate_kernel.)
static constexpr int kTileRecWords = 32;
static std::vector<uint32_t> tile_records(const std::vector<int4>& tiles, const std::vector<int2>& ents) {
  std::vector<uint32_t> rec(tiles.size() * kTileRecWords, 0u);
  for (size_t t = 0; t < tiles.size(); ++t) {
    uint32_t* r = rec.data() + t * kTileRecWords;
    uint32_t start = 0;
    for (int32_t e = tiles[t].z; e < tiles[t].w; ++e) {
      start |= 1u << ((ents[e].y >> 16) / 16);
      r[16 + (e - tiles[t].z)] = (uint32_t)ents[e].x;
    }
    r[0] = (uint32_t)tiles[t].y | ((uint32_t)(tiles[t].w - tiles[t].z) << 16);
    r[1] = start | (0xFFFFu & ~((1u << (tiles[t].y / 16)) - 1u));  // groups past n_rows: own "chunks"
    r[4] = (uint32_t)tiles[t].x;
  }
  return rec;
}

extern "C" hiper_status hiper_pack_plan(const int32_t* lens, int64_t n, int32_t* tiles_out,
                                        int32_t* ents_out, int64_t* n_tiles, int64_t* n_rows) {
  if (n < 0) return fail(HIPER_ERR_INVALID_ARG, "n < 0");
  if (n > 0 && (!lens || !tiles_out || !ents_out)) return fail(HIPER_ERR_INVALID_ARG, "NULL array");
  if (n > 0x7FFFFFFFll) return fail(HIPER_ERR_UNSUPPORTED, "n >= 2^31");
  std::vector<int4> tiles;
  std::vector<int2> ents;
  std::vector<int64_t> dst;
  int64_t rows = 0;
  TRY(pack_plan(lens, n, tiles, ents, dst, rows));
  if (n > 0) {
    memcpy(tiles_out, tiles.data(), tiles.size() * sizeof(int4));
    memcpy(ents_out, ents.data(), ents.size() * sizeof(int2));
  }
  if (n_tiles) *n_tiles = (int64_t)tiles.size();
  if (n_rows) *n_rows = rows;
  return HIPER_OK;
}

// dim % 16 == 0 (one MMA K step; the TMA boxes are 64 wide and zero-fill the columns past dim).
// Token path: dim <= 256.  Pooled path (HIPER_POOLED, one row per item, a12): dim <= 4096.
static constexpr int32_t kMaxTokenDim = 256, kMaxPooledDim = 4096;
static hiper_status check_dims(int32_t dim, bool pooled = false) {
  if (dim <= 0) return fail(HIPER_ERR_INVALID_ARG, "dim must be positive (got %d)", dim);
  const int32_t mx = pooled ? kMaxPooledDim : kMaxTokenDim;
  if (dim % 16 != 0 || dim > mx)
    return fail(HIPER_ERR_UNSUPPORTED, "%s dim %d unsupported (multiple of 16, <= %d)",
                pooled ? "pooled" : "token", dim, mx);
  return HIPER_OK;
}
static inline int32_t num_kb_of(int32_t dim) { return (dim + 63) / 64; }

static hiper_status launch_norm(const void* in, hiper_dtype dtype, int64_t n_src, int32_t in_rows,
                                const int32_t* lens_dev, int64_t n_items, int32_t out_rows,
                                int32_t dim, uint32_t flags, __nv_bfloat16* out, uint32_t* status,
                                cudaStream_t stream, const int64_t* dst_row = nullptr) {
  const int64_t rows = n_items * (int64_t)out_rows;
  if (rows == 0) return HIPER_OK;
  const int threads = 256;
  const uint32_t an = (flags & HIPER_ASSUME_NORMALIZED) ? 1u : 0u;
  const uint32_t cf = (flags & HIPER_CHECK_FINITE) ? 1u : 0u;
  if (dim == 64 || dim == 128 || dim == 256) {  // d/16 threads per row: coalesced, same fma order
    const int tpr = dim / 16;
    const int64_t blocks = (rows * tpr + threads - 1) / threads;
    if (blocks > 0x7FFFFFFF) return fail(HIPER_ERR_UNSUPPORTED, "too many rows");
#define HIPER_NORM_TPR(T, TPR)                                                                       \
  norm_layout_tpr_kernel<T, TPR><<<(unsigned)blocks, threads, 0, stream>>>(                          \
      (const T*)in, n_src, in_rows, lens_dev, n_items, out_rows, dim, an, cf, out, status, dst_row)
    if (dtype == HIPER_F32) {
      if (tpr == 4) HIPER_NORM_TPR(float, 4); else if (tpr == 8) HIPER_NORM_TPR(float, 8); else HIPER_NORM_TPR(float, 16);
    } else {
      if (tpr == 4) HIPER_NORM_TPR(__nv_bfloat16, 4); else if (tpr == 8) HIPER_NORM_TPR(__nv_bfloat16, 8); else HIPER_NORM_TPR(__nv_bfloat16, 16);
    }
#undef HIPER_NORM_TPR
    CUDA_TRY(cudaGetLastError());
    ++g_launches;
    return HIPER_OK;
  }
  if (dst_row != nullptr && in == (const void*)out)
    return fail(HIPER_ERR_UNSUPPORTED, "in-place packed layout needs dim 64, 128 or 256");
  const int64_t blocks = (rows + threads - 1) / threads;
  if (blocks > 0x7FFFFFFF) return fail(HIPER_ERR_UNSUPPORTED, "too many rows");
  if (dtype == HIPER_F32)
    norm_layout_kernel<float><<<(unsigned)blocks, threads, 0, stream>>>(
        (const float*)in, n_src, in_rows, lens_dev, n_items, out_rows, dim, an, cf, out, status,
        dst_row);
  else
    norm_layout_kernel<__nv_bfloat16><<<(unsigned)blocks, threads, 0, stream>>>(
        (const __nv_bfloat16*)in, n_src, in_rows, lens_dev, n_items, out_rows, dim, an, cf, out,
        status, dst_row);
  CUDA_TRY(cudaGetLastError());
  ++g_launches;
  return HIPER_OK;
}

// Query and document layouts of one ColTrast step in a single launch (norm_layout2_kernel).
static hiper_status launch_norm2(const void* in_a, int64_t n_a, int32_t in_rows_a, const int32_t* lens_a,
                                 int64_t items_a, int32_t out_rows_a, __nv_bfloat16* out_a,
                                 const void* in_b, int64_t n_b, int32_t in_rows_b, const int32_t* lens_b,
                                 int64_t items_b, int32_t out_rows_b, __nv_bfloat16* out_b,
                                 hiper_dtype dtype, int32_t dim, uint32_t flags, uint32_t* status,
                                 cudaStream_t stream) {
  const int threads = 256;
  if (dim != 64 && dim != 128 && dim != 256) {  // other dims: the one-thread-per-row kernel, twice
    TRY(launch_norm(in_a, dtype, n_a, in_rows_a, lens_a, items_a, out_rows_a, dim, flags, out_a, status, stream));
    return launch_norm(in_b, dtype, n_b, in_rows_b, lens_b, items_b, out_rows_b, dim, flags, out_b, status, stream);
  }
  const int tpr = dim / 16;
  const int64_t ba = (items_a * out_rows_a * tpr + threads - 1) / threads;
  const int64_t bb = (items_b * out_rows_b * tpr + threads - 1) / threads;
  if (ba + bb == 0) return HIPER_OK;
  if (ba + bb > 0x7FFFFFFF) return fail(HIPER_ERR_UNSUPPORTED, "too many rows");
  const NormSeg a{in_a, n_a, in_rows_a, lens_a, items_a, out_rows_a, out_a};
  const NormSeg b{in_b, n_b, in_rows_b, lens_b, items_b, out_rows_b, out_b};
  const uint32_t an = (flags & HIPER_ASSUME_NORMALIZED) ? 1u : 0u;
  const uint32_t cf = (flags & HIPER_CHECK_FINITE) ? 1u : 0u;
#define HIPER_NORM2(T, TPR) \
  norm_layout2_kernel<T, TPR><<<(unsigned)(ba + bb), threads, 0, stream>>>(a, b, ba, dim, an, cf, status)
  if (dtype == HIPER_F32) {
    if (tpr == 4) HIPER_NORM2(float, 4); else if (tpr == 8) HIPER_NORM2(float, 8); else HIPER_NORM2(float, 16);
  } else {
    if (tpr == 4) HIPER_NORM2(__nv_bfloat16, 4); else if (tpr == 8) HIPER_NORM2(__nv_bfloat16, 8); else HIPER_NORM2(__nv_bfloat16, 16);
  }
#undef HIPER_NORM2
  CUDA_TRY(cudaGetLastError());
  ++g_launches;
  return HIPER_OK;
}

static hiper_status check_lens(const int32_t* lens, int64_t n, int32_t max_len, const char* what) {
  if (n > 0 && lens == nullptr) return fail(HIPER_ERR_INVALID_ARG, "%s lens is NULL", what);
  for (int64_t i = 0; i < n; ++i) {
    if (lens[i] == 0) return fail(HIPER_ERR_EMPTY_TOKENS, "%s %lld has 0 tokens", what, (long long)i);
    if (lens[i] < 0 || lens[i] > max_len)
      return fail(HIPER_ERR_INVALID_ARG, "%s %lld length %d outside 1..%d", what, (long long)i,
                  lens[i], max_len);
  }
  return HIPER_OK;
}

extern "C" hiper_status hiper_index_build(const void* tokens, hiper_dtype dtype, const int32_t* lens,
                                          int64_t n, int32_t max_len, int32_t dim, int64_t id_base,
                                          uint32_t flags, hiper_stream_t stream_, hiper_index** out) {
  g_launches = 0;
  HiperRange nv("hiper_index_build");
  cudaStream_t stream = (cudaStream_t)stream_;
  if (!out) return fail(HIPER_ERR_INVALID_ARG, "out is NULL");
  *out = nullptr;
  if (n < 0) return fail(HIPER_ERR_INVALID_ARG, "n < 0");
  if (dtype != HIPER_F32 && dtype != HIPER_BF16) return fail(HIPER_ERR_INVALID_ARG, "bad dtype");
  if (flags & ~(uint32_t)(HIPER_ASSUME_NORMALIZED | HIPER_CHECK_FINITE | HIPER_BORROW_TOKENS |
                          HIPER_PACKED | HIPER_POOLED))
    return fail(HIPER_ERR_INVALID_ARG, "unknown flags 0x%x", flags);
  if (max_len < 1) return fail(HIPER_ERR_INVALID_ARG, "max_len must be >= 1");
  if (max_len > kMaxChunkLen) return fail(HIPER_ERR_UNSUPPORTED, "max_len %d > %d", max_len, kMaxChunkLen);
  const bool pooled = (flags & HIPER_POOLED) != 0;  // the pooled limit case (a12)
  if (pooled && (max_len != 1 || (flags & HIPER_PACKED)))
    return fail(HIPER_ERR_INVALID_ARG, "HIPER_POOLED takes one vector per item (max_len 1, not packed)");
  TRY(check_dims(dim, pooled));
  if (id_base < 0 || id_base + n >= 0xFFFFFFFFll)
    return fail(HIPER_ERR_UNSUPPORTED, "global ids must be < 2^32-1");
  const bool packed = (flags & HIPER_PACKED) != 0;
  const int32_t ld_pad = pooled ? 1 : (int32_t)round_up(max_len, 16);
  if (!packed && n * ld_pad >= 0x7FFFFFFFll)
    return fail(HIPER_ERR_UNSUPPORTED, "n * ld_pad >= 2^31 rows for one index; shard the corpus");
  TRY(check_lens(lens, n, max_len, "chunk"));
  const bool borrow = (flags & HIPER_BORROW_TOKENS) != 0;
  if (packed && borrow && dtype != HIPER_BF16)
    return fail(HIPER_ERR_INVALID_ARG, "HIPER_PACKED | HIPER_BORROW_TOKENS needs bf16 packed tokens");
  if (packed && borrow && dim != 64 && dim != 128 && dim != 256)
    return fail(HIPER_ERR_UNSUPPORTED, "in-place packed layout needs dim 64, 128 or 256");
  std::vector<int4> p_tiles;
  std::vector<int2> p_ents;
  std::vector<int64_t> p_dst;
  int64_t p_rows = 0;
  if (packed) TRY(pack_plan(lens, n, p_tiles, p_ents, p_dst, p_rows));
  if (borrow && !packed && (dtype != HIPER_BF16 || max_len != ld_pad || (dim % 8) != 0))
    return fail(HIPER_ERR_INVALID_ARG, "HIPER_BORROW_TOKENS needs bf16 tokens and max_len %% 16 == 0");
  if (n > 0) {
    if (!tokens) return fail(HIPER_ERR_INVALID_ARG, "tokens is NULL");
    if (((uintptr_t)tokens & 15) != 0) return fail(HIPER_ERR_INVALID_ARG, "tokens must be 16-B aligned");
    if (!is_device_ptr(tokens)) return fail(HIPER_ERR_INVALID_ARG, "tokens must be device memory");
  }
  DevInfo di;
  TRY(device_info(di));

  hiper_index_s* ix = new hiper_index_s();
  ix->n = n;
  ix->max_len = max_len;
  ix->ld_pad = ld_pad;
  ix->dim = dim;
  ix->id_base = id_base;
  ix->device = di.device;
  ix->pooled = pooled;
  int64_t* dst_dev = nullptr;
  auto cleanup = [&](hiper_status s) {
    if (ix->owns_tok && ix->tok) cudaFree(ix->tok);
    if (ix->lens) cudaFree(ix->lens);
    if (ix->tiles) cudaFree(ix->tiles);
    if (ix->recs) cudaFree(ix->recs);
    if (ix->ents) cudaFree(ix->ents);
    if (dst_dev) cudaFree(dst_dev);
    ix->row_of = nullptr;
    delete ix;
    return s;
  };
  const int64_t n_alloc = std::max<int64_t>(n, 1);
  if (cudaMalloc(&ix->lens, n_alloc * sizeof(int32_t)) != cudaSuccess)
    return cleanup(fail(HIPER_ERR_OUT_OF_MEMORY, "lens alloc"));
  if (borrow && !packed) {
    ix->tok = (__nv_bfloat16*)const_cast<void*>(tokens);
  } else if (packed) {
    ix->packed = true;
    ix->n_tiles = (int64_t)p_tiles.size();
    ix->n_rows = p_rows;
    if (borrow) {  // the caller's buffer already has the hiper_pack_plan layout: NORM in place
      ix->tok = (__nv_bfloat16*)const_cast<void*>(tokens);
    } else {
      if (cudaMalloc(&ix->tok, (size_t)std::max<int64_t>(p_rows, 1) * dim * 2) != cudaSuccess)
        return cleanup(fail(HIPER_ERR_OUT_OF_MEMORY, "packed layout alloc %lld bytes", (long long)p_rows * dim * 2));
      ix->owns_tok = true;
    }
    const std::vector<uint32_t> p_rec = tile_records(p_tiles, p_ents);
    if (cudaMalloc(&ix->recs, std::max<size_t>(p_rec.size(), 1) * sizeof(uint32_t)) != cudaSuccess ||
        (n > 0 && cudaMemcpyAsync(ix->recs, p_rec.data(), p_rec.size() * sizeof(uint32_t), cudaMemcpyHostToDevice, stream) != cudaSuccess))
      return cleanup(fail(HIPER_ERR_OUT_OF_MEMORY, "tile records"));
    if (cudaMalloc(&ix->tiles, std::max<size_t>(p_tiles.size(), 1) * sizeof(int4)) != cudaSuccess ||
        cudaMalloc(&ix->ents, std::max<size_t>(p_ents.size(), 1) * sizeof(int2)) != cudaSuccess ||
        cudaMalloc(&dst_dev, std::max<size_t>(p_dst.size(), 1) * sizeof(int64_t)) != cudaSuccess)
      return cleanup(fail(HIPER_ERR_OUT_OF_MEMORY, "packing tables"));
    if (n > 0 &&
        (cudaMemcpyAsync(ix->tiles, p_tiles.data(), p_tiles.size() * sizeof(int4), cudaMemcpyHostToDevice, stream) != cudaSuccess ||
         cudaMemcpyAsync(ix->ents, p_ents.data(), p_ents.size() * sizeof(int2), cudaMemcpyHostToDevice, stream) != cudaSuccess ||
         cudaMemcpyAsync(dst_dev, p_dst.data(), p_dst.size() * sizeof(int64_t), cudaMemcpyHostToDevice, stream) != cudaSuccess))
      return cleanup(fail(HIPER_ERR_CUDA, "packing tables copy"));
  } else {
    if (cudaMalloc(&ix->tok, (size_t)n_alloc * ld_pad * dim * 2) != cudaSuccess)
      return cleanup(fail(HIPER_ERR_OUT_OF_MEMORY, "layout alloc %lld bytes",
                          (long long)n_alloc * ld_pad * dim * 2));
    ix->owns_tok = true;
  }
  uint32_t* status = nullptr;
  if (cudaMalloc(&status, sizeof(uint32_t)) != cudaSuccess)
    return cleanup(fail(HIPER_ERR_OUT_OF_MEMORY, "status alloc"));
  hiper_status st = HIPER_OK;
  uint32_t hstat = 0;
  do {
    if (cudaMemsetAsync(status, 0, sizeof(uint32_t), stream) != cudaSuccess) { st = fail(HIPER_ERR_CUDA, "memset"); break; }
    if (n > 0 && cudaMemcpyAsync(ix->lens, lens, n * sizeof(int32_t), cudaMemcpyHostToDevice, stream) != cudaSuccess) {
      st = fail(HIPER_ERR_CUDA, "lens copy"); break;
    }
    st = launch_norm(tokens, dtype, n, max_len, ix->lens, n, ld_pad, dim,
                     flags | HIPER_CHECK_FINITE, ix->tok, status, stream, dst_dev);
    if (st != HIPER_OK) break;
    if (packed && n > 0) {  // padding rows repeat each chunk's last row (unmasked packed epilogue)
      const int64_t threads = (int64_t)n * (dim / 8);
      pack_pad_replicate_kernel<<<(unsigned)((threads + 255) / 256), 256, 0, stream>>>(
          ix->tok, dst_dev, ix->lens, n, dim);
      if (cudaGetLastError() != cudaSuccess) { st = fail(HIPER_ERR_CUDA, "pad replicate launch"); break; }
      ++g_launches;
    }
    if (cudaMemcpyAsync(&hstat, status, sizeof(uint32_t), cudaMemcpyDeviceToHost, stream) != cudaSuccess ||
        cudaStreamSynchronize(stream) != cudaSuccess) {
      st = fail(HIPER_ERR_CUDA, "build sync: %s", cudaGetErrorString(cudaGetLastError()));
      break;
    }
    if (hstat & kStatusNonFinite) { st = fail(HIPER_ERR_NONFINITE, "chunk tokens contain non-finite values"); break; }
    if (hstat & kStatusZeroRow) { st = fail(HIPER_ERR_ZERO_VECTOR, "a chunk token row has norm 0"); break; }
    if (n > 0 && pooled) {
      st = make_tmap(&ix->tmap, ix->tok, n, dim, 128);  // pooled kernel: 128 chunk rows per CTA
    } else if (n > 0 && packed) {
      // half a full tile per CTA; a shorter tile's MMA reads only its first n_rows/2 rows
      st = make_tmap(&ix->tmap_half, ix->tok, p_rows, dim, kTileRows / 2);
    } else if (n > 0) {
      // this CTA's rows of a chunk: ld_pad / 2, or 128 of each 256-row half when ld_pad > 256
      st = make_tmap(&ix->tmap_half, ix->tok, n * (int64_t)ld_pad, dim, ld_pad > 256 ? 128 : ld_pad / 2);
    }
  } while (0);
  cudaFree(status);
  if (st != HIPER_OK) return cleanup(st);
  ix->row_of = dst_dev;  // kept: stage 2 of hiper_two_stage_topk reads packed chunks by id
  *out = ix;
  return HIPER_OK;
}

extern "C" hiper_status hiper_index_destroy(hiper_index* ix) {
  if (!ix) return HIPER_OK;
  if (ix->owns_tok && ix->tok) cudaFree(ix->tok);
  if (ix->lens) cudaFree(ix->lens);
  if (ix->tiles) cudaFree(ix->tiles);
  if (ix->recs) cudaFree(ix->recs);
  if (ix->ents) cudaFree(ix->ents);
  if (ix->row_of) cudaFree(ix->row_of);
  delete ix;
  return HIPER_OK;
}

extern "C" hiper_status hiper_index_info(const hiper_index* ix, int64_t* n, int32_t* max_len,
                                         int32_t* dim, int32_t* ld_pad, int64_t* id_base,
                                         const void** layout, const int32_t** lens_dev) {
  if (!ix) return fail(HIPER_ERR_INVALID_ARG, "index is NULL");
  if (n) *n = ix->n;
  if (max_len) *max_len = ix->max_len;
  if (dim) *dim = ix->dim;
  if (ld_pad) *ld_pad = ix->ld_pad;
  if (id_base) *id_base = ix->id_base;
  if (layout) *layout = ix->tok;
  if (lens_dev) *lens_dev = ix->lens;
  return HIPER_OK;
}

extern "C" hiper_status hiper_index_pack_info(const hiper_index* ix, int32_t* packed, int64_t* n_tiles,
                                              int64_t* n_rows, const void** tiles_dev,
                                              const void** ents_dev) {
  if (!ix) return fail(HIPER_ERR_INVALID_ARG, "index is NULL");
  if (packed) *packed = ix->packed ? 1 : 0;
  if (n_tiles) *n_tiles = ix->n_tiles;
  if (n_rows) *n_rows = ix->n_rows;
  if (tiles_dev) *tiles_dev = ix->tiles;
  if (ents_dev) *ents_dev = ix->ents;
  return HIPER_OK;
}

// ============================================================================ query preparation
// A query occupies QS = 32, 64 or 128 padded token rows (q_max_len <= 32 / 64 / 128): one, two or
// four warps of TMEM lanes.  Queries are padded to fill whole CTA pairs: M = 256 rows = 256 / QS.
static int32_t qs_of(int32_t q_max_len) { return q_max_len <= 32 ? 32 : (q_max_len <= 64 ? 64 : 128); }
static int32_t n_q_pad_of(int32_t n_q, int32_t qs = 32) {
  return (int32_t)round_up(std::max(n_q, 1), 256 / qs);
}
// Query layout bytes for any q_max_len (the workspace-size entry points do not take q_max_len).
static size_t q_layout_bytes_max(int32_t n_q, int32_t dim) {
  size_t m = 0;
  for (int32_t qs = 32; qs <= 128; qs *= 2) m = std::max(m, (size_t)n_q_pad_of(n_q, qs) * qs * dim * 2);
  return m;
}

static hiper_status validate_queries(const void* q_tokens, hiper_dtype dtype, const int32_t* q_lens,
                                     int32_t n_q, int32_t q_max_len, int32_t dim, uint32_t flags,
                                     bool pooled = false) {
  if (dtype != HIPER_F32 && dtype != HIPER_BF16) return fail(HIPER_ERR_INVALID_ARG, "bad dtype");
  if (n_q < 0) return fail(HIPER_ERR_INVALID_ARG, "n_q < 0");
  if (flags & ~(uint32_t)(HIPER_ASSUME_NORMALIZED | HIPER_CHECK_FINITE | HIPER_VALIDATE_SYNC))
    return fail(HIPER_ERR_INVALID_ARG, "unknown flags 0x%x", flags);
  TRY(check_dims(dim, pooled));
  if (pooled && q_max_len != 1)
    return fail(HIPER_ERR_UNSUPPORTED, "a pooled index (HIPER_POOLED) takes pooled queries (q_max_len 1)");
  if (q_max_len < 1) return fail(HIPER_ERR_INVALID_ARG, "q_max_len must be >= 1");
  if (q_max_len > kMaxQueryLen) return fail(HIPER_ERR_UNSUPPORTED, "q_max_len %d > %d", q_max_len, kMaxQueryLen);
  TRY(check_lens(q_lens, n_q, q_max_len, "query"));
  if (n_q > 0) {
    if (!q_tokens) return fail(HIPER_ERR_INVALID_ARG, "q_tokens is NULL");
    if (((uintptr_t)q_tokens & 15) != 0) return fail(HIPER_ERR_INVALID_ARG, "q_tokens must be 16-B aligned");
    if (!is_device_ptr(q_tokens)) return fail(HIPER_ERR_INVALID_ARG, "q_tokens must be device memory");
  }
  return HIPER_OK;
}

// Device-side query prep: q_lens HOST -> lens_dev (staged), NORM into layout [n_q_pad][QS][dim].
static hiper_status prep_queries(const void* q_tokens, hiper_dtype dtype, const int32_t* q_lens,
                                 int32_t n_q, int32_t q_max_len, int32_t dim, uint32_t flags,
                                 int32_t* lens_dev, __nv_bfloat16* layout, uint32_t* status,
                                 cudaStream_t stream) {
  TRY(stage_h2d(lens_dev, q_lens, (size_t)n_q * sizeof(int32_t), stream));
  const int32_t qs = qs_of(q_max_len);
  return launch_norm(q_tokens, dtype, n_q, q_max_len, lens_dev, n_q_pad_of(n_q, qs), qs, dim, flags,
                     layout, status, stream);
}

static hiper_status sync_status(const uint32_t* status, cudaStream_t stream) {
  uint32_t h = 0;
  CUDA_TRY(cudaMemcpyAsync(&h, status, sizeof(h), cudaMemcpyDeviceToHost, stream));
  CUDA_TRY(cudaStreamSynchronize(stream));
  if (h & kStatusNonFinite) return fail(HIPER_ERR_NONFINITE, "a query row is non-finite");
  if (h & kStatusZeroRow) return fail(HIPER_ERR_ZERO_VECTOR, "a real query row has norm 0");
  return HIPER_OK;
}

extern "C" hiper_status hiper_prepare_queries(const void* q_tokens, hiper_dtype dtype,
                                              const int32_t* q_lens, int32_t n_q, int32_t q_max_len,
                                              int32_t dim, uint32_t flags, void* out_layout,
                                              uint32_t* status, hiper_stream_t stream_) {
  g_launches = 0;
  HiperRange nv("hiper_prepare_queries");
  cudaStream_t stream = (cudaStream_t)stream_;
  TRY(validate_queries(q_tokens, dtype, q_lens, n_q, q_max_len, dim, flags));
  if (!out_layout || !is_device_ptr(out_layout)) return fail(HIPER_ERR_INVALID_ARG, "out_layout must be device memory");
  DevInfo di;
  TRY(device_info(di));
  int32_t* lens_dev = nullptr;
  CUDA_TRY(cudaMallocAsync(&lens_dev, std::max(n_q, 1) * sizeof(int32_t), stream));
  hiper_status st = prep_queries(q_tokens, dtype, q_lens, n_q, q_max_len, dim, flags, lens_dev,
                                 (__nv_bfloat16*)out_layout, status, stream);
  cudaFreeAsync(lens_dev, stream);
  return st;
}

// ============================================================================ the MaxSim kernel launch
static int32_t choose_parts(int32_t n_groups, int64_t n_chunks, int num_sms) {
  if (n_chunks <= 0) return 0;
  const int64_t p0 = num_sms / std::gcd(n_groups, num_sms);
  return (int32_t)std::max<int64_t>(1, std::min<int64_t>(p0, n_chunks));
}

// Top-k path: L2 bands.  Units are (row group, corpus partition), ordered partition-major, and a wave
// of resident pairs covers at most two consecutive partitions.  With partitions of ~kBandBytes of
// corpus, both stay resident in the 126 MB L2 while every row group streams them, so HBM reads the
// corpus ~once per query batch (37 partitions at config 3 re-read it 2.7x).  The partition count is
// a multiple of p0 (full waves) and is capped so the per-(partition, group) top-k lists stay small.
// HIPER_BAND_MB overrides the band size (0 = the minimal partition count).
static int64_t band_bytes() {
  static const int64_t b = [] {
    const char* e = getenv("HIPER_BAND_MB");
    return e ? (int64_t)atoll(e) << 20 : (int64_t)24 << 20;
  }();
  return b;
}
static int32_t choose_parts_topk(int32_t n_groups, int64_t n_slots, int num_slots, int64_t slot_bytes,
                                 int32_t n_q_pad, int32_t k) {
  if (n_slots <= 0) return 0;
  const int64_t p0 = num_slots / std::gcd(n_groups, num_slots);
  int64_t p = p0;
  if (band_bytes() > 0) {
    const int64_t want = (n_slots * slot_bytes + band_bytes() - 1) / band_bytes();
    p = std::max<int64_t>(p0, (want + p0 - 1) / p0 * p0);
    const int64_t cap = ((int64_t)512 << 20) / ((int64_t)kEpiGroups * n_q_pad * k * 8);
    p = std::min<int64_t>(p, std::max<int64_t>(p0, cap / p0 * p0));
  }
  return (int32_t)std::max<int64_t>(1, std::min<int64_t>(p, n_slots));
}

// The MaxSim kernel is the CTA-pair kernel (cta_group::2, M = 256 query-token rows per pair).
struct KernelPlan {
  int32_t qs = 32, qw = 1, h = 1;  // query slot rows, warps per query, MMA halves per chunk
  int32_t qpg = 8;                 // queries per row group (256 / qs)
  int32_t n_q_pad = 0, n_groups = 0, n_parts = 0, n_stages = 0, a_bufs = 2;
  uint32_t a_bytes = 0, stage_bytes = 0, box_rows = 0, smem_bytes = 0;
  int grid = 0;
};

// slot_rows: token rows per kernel slot (a chunk's ld_pad, or 256 for a packed tile).
static hiper_status plan_kernel(const DevInfo& di, int32_t n_q, int32_t q_max_len, int64_t n_slots,
                                int32_t slot_rows, int32_t dim, KernelPlan& kp, int32_t topk_k = 0) {
  kp.qs = qs_of(q_max_len);
  kp.qw = kp.qs / 32;
  kp.qpg = 256 / kp.qs;
  kp.h = slot_rows > 256 ? 2 : 1;
  const int slots = di.num_sms / 2;  // CTA pairs
  kp.n_q_pad = n_q_pad_of(n_q, kp.qs);
  kp.n_groups = kp.n_q_pad / kp.qpg;
  kp.n_parts = topk_k > 0 ? choose_parts_topk(kp.n_groups, n_slots, slots, (int64_t)slot_rows * dim * 2,
                                              kp.n_q_pad, topk_k)
                          : choose_parts(kp.n_groups, n_slots, slots);
  const uint32_t nkb = (uint32_t)num_kb_of(dim);
  kp.a_bytes = nkb * 16384u;
  // one stage = this CTA's rows of one chunk (half): ld_pad / 2, or 128 of a 256-row half
  kp.box_rows = kp.h == 2 ? 128u : (uint32_t)slot_rows / 2;
  kp.stage_bytes = kp.box_rows * 128u * nkb;
  // The A tile is double-buffered across units unless one buffer buys an extra B stage on long
  // units: a unit boundary then costs one A load (~1 us), while the extra stage hides L2 latency and
  // lockstep pauses on every chunk (config3, same box: 5 -> 6 stages, 633 -> 646 q/s,
  // profiles/r02/ablation/one_a_buffer.txt).  Large dims fall back to one buffer anyway.
  auto stages_for = [&](int32_t bufs, uint32_t& smem) {
    const uint32_t fixed = 1024u /*align slack*/ + bufs * kp.a_bytes + 2048u /*barriers, ring, sums*/;
    const uint32_t avail = (uint32_t)di.max_smem > fixed ? (uint32_t)di.max_smem - fixed : 0u;
    const int32_t st = (int32_t)std::min<uint32_t>(12u, avail / kp.stage_bytes);
    smem = fixed + (uint32_t)st * kp.stage_bytes;
    return st;
  };
  uint32_t smem1 = 0, smem2 = 0;
  const int32_t st1 = stages_for(1, smem1), st2 = stages_for(2, smem2);
  const bool long_units = kp.n_parts > 0 && n_slots / kp.n_parts >= 64;
  static const char* force = getenv("HIPER_A_BUFS");  // ablation: force 1 or 2
  const bool one = force ? force[0] == '1' : (st2 < 2 || (long_units && st1 > st2));
  kp.a_bufs = one ? 1 : 2;
  kp.n_stages = one ? st1 : st2;
  kp.smem_bytes = one ? smem1 : smem2;
  if (kp.n_stages < 2) return fail(HIPER_ERR_UNSUPPORTED, "not enough shared memory for 2 stages");
  const int64_t units = (int64_t)kp.n_groups * kp.n_parts;
  kp.grid = (int)std::min<int64_t>(units, slots) * 2;
  return HIPER_OK;
}

// The kernel arguments every MaxSim launch shares (plan + query side + the index's slots).
static MaxsimArgs maxsim_args(const KernelPlan& kp, int32_t n_q, int64_t n_slots, int32_t ld_pad,
                              int32_t dim, const int32_t* qlens_dev, const int32_t* dlens_dev) {
  MaxsimArgs a{};
  a.n_q = n_q;
  a.n_groups = kp.n_groups;
  a.n_parts = kp.n_parts;
  a.ld_pad = ld_pad;
  a.num_kb = num_kb_of(dim);
  a.k = 1;
  a.n_stages = kp.n_stages;
  a.a_bytes = kp.a_bytes;
  a.stage_bytes = kp.stage_bytes;
  a.box_rows = kp.box_rows;
  a.a_bufs = kp.a_bufs;
  a.q_pad = kp.n_q_pad;
  a.n_chunks = n_slots;
  a.q_lens = qlens_dev;
  a.d_lens = dlens_dev;
  return a;
}

// ---------------------------------------------------------------------------- live kernel timing
// Every launch of a hot kernel is bracketed by CUDA events on its own stream while profiling is on;
// records carry the kernel class (hiper.h HIPER_PROF_*) so a step with several hot kernels (the
// two-stage search) reports each one's share.
namespace {
struct ProfEv {
  cudaEvent_t a, b;
  int32_t tag;
};
struct ProfileRec {
  std::mutex mu;
  bool on = false;
  std::vector<ProfEv> live;
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> pool;
};
ProfileRec g_prof;
}  // namespace

extern "C" void hiper_profile_enable(int32_t on) {
  std::lock_guard<std::mutex> lock(g_prof.mu);
  g_prof.on = on != 0;
}

// tag < 0: every kernel class.  Reads (synchronising on the events) and forgets the matching records.
static hiper_status profile_read(int32_t tag, double* ms, int32_t* n_launches) {
  std::lock_guard<std::mutex> lock(g_prof.mu);
  double total = 0.0;
  int32_t n = 0;
  std::vector<ProfEv> keep;
  for (auto& e : g_prof.live) {
    if (tag >= 0 && e.tag != tag) {
      keep.push_back(e);
      continue;
    }
    CUDA_TRY(cudaEventSynchronize(e.b));
    float t = 0.f;
    CUDA_TRY(cudaEventElapsedTime(&t, e.a, e.b));
    total += t;
    ++n;
    g_prof.pool.push_back({e.a, e.b});
  }
  g_prof.live.swap(keep);
  if (ms) *ms = total;
  if (n_launches) *n_launches = n;
  return HIPER_OK;
}
extern "C" hiper_status hiper_profile_read(double* maxsim_ms, int32_t* n_launches) {
  return profile_read(-1, maxsim_ms, n_launches);
}
extern "C" hiper_status hiper_profile_read_tagged(int32_t tag, double* ms, int32_t* n_launches) {
  return profile_read(tag, ms, n_launches);
}

struct ProfTicket {
  cudaEvent_t a = nullptr, b = nullptr;
  int32_t tag = 0;
  bool rec = false;
};
static hiper_status profile_begin(cudaStream_t stream, int32_t tag, ProfTicket* t) {
  std::lock_guard<std::mutex> lock(g_prof.mu);
  t->rec = g_prof.on;
  t->tag = tag;
  if (!g_prof.on) return HIPER_OK;
  if (g_prof.pool.empty()) {
    cudaEvent_t a, b;
    CUDA_TRY(cudaEventCreate(&a));
    CUDA_TRY(cudaEventCreate(&b));
    g_prof.pool.push_back({a, b});
  }
  t->a = g_prof.pool.back().first;
  t->b = g_prof.pool.back().second;
  g_prof.pool.pop_back();
  CUDA_TRY(cudaEventRecord(t->a, stream));
  return HIPER_OK;
}

static hiper_status profile_end(cudaStream_t stream, const ProfTicket& t) {
  if (!t.rec) return HIPER_OK;
  CUDA_TRY(cudaEventRecord(t.b, stream));
  std::lock_guard<std::mutex> lock(g_prof.mu);
  g_prof.live.push_back({t.a, t.b, t.tag});
  return HIPER_OK;
}

static int debug_mode() {
  static const int m = [] {
    const char* e = getenv("HIPER_DEBUG_MODE");
    return e ? atoi(e) : 0;
  }();
  return m;
}

template <int MODE, int KR, bool PACKED, int QW, int H>
static hiper_status launch_maxsim_t(const KernelPlan& kp, const CUtensorMap& tq, const CUtensorMap& td,
                                    const MaxsimArgs& a, cudaStream_t stream) {
  ProfTicket ev;
  static const bool stats_on = getenv("HIPER_PIPE_STATS") != nullptr;
  // production: no instrumentation compiled in; HIPER_PIPE_STATS / HIPER_DEBUG_MODE select the
  // instrumented (STATS) instantiations
  auto kern = stats_on ? maxsim_sm100_pair_kernel<MODE, KR, 0, PACKED, true, QW, H>
                       : maxsim_sm100_pair_kernel<MODE, KR, 0, PACKED, false, QW, H>;
  if constexpr (!PACKED && MODE == 1 && KR == 1 && QW == 1 && H == 1) {
    if (debug_mode() == 1) kern = maxsim_sm100_pair_kernel<MODE, KR, 1, false, true>;
    if (debug_mode() == 2) kern = maxsim_sm100_pair_kernel<MODE, KR, 2, false, true>;
    if (debug_mode() == 3) kern = maxsim_sm100_pair_kernel<MODE, KR, 3, false, true>;
    if (debug_mode() == 4) kern = maxsim_sm100_pair_kernel<MODE, KR, 4, false, true>;
  }
  CUDA_TRY(set_max_smem((const void*)kern, (int)kp.smem_bytes));
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)kp.grid);
  cfg.blockDim = dim3(kMaxsimThreads);
  cfg.dynamicSmemBytes = kp.smem_bytes;
  cfg.stream = stream;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  // programmatic dependent launch: the kernel's set-up (barriers, TMEM, tensor-map prefetch)
  // overlaps the previous kernel's tail; it waits (griddepcontrol.wait) before reading its inputs
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 2;
  unsigned long long* st = nullptr;
  MaxsimArgs b = a;
  static const bool late = getenv("HIPER_LATE_RELEASE") && getenv("HIPER_LATE_RELEASE")[0] == '1';
  b.late_release = late ? 1 : 0;
  static const int32_t ls_every = [] {  // lockstep publish / check interval in chunks (ablation knob)
    const char* e = getenv("HIPER_LOCKSTEP_EVERY");
    int v = e ? atoi(e) : 256;  // 16 -> 256: +2-3% at config 3 (ablation/lockstep_r02.txt)
    int p = 1;
    while (p < v && p < 1024) p <<= 1;
    return p;
  }();
  b.ls_mask = ls_every - 1;
  if (stats_on) {
    CUDA_TRY(cudaMalloc(&st, 8 * sizeof(unsigned long long)));
    CUDA_TRY(cudaMemsetAsync(st, 0, 8 * sizeof(unsigned long long), stream));
    b.stats = st;
  }
  TRY(profile_begin(stream, HIPER_PROF_MAXSIM, &ev));
  CUDA_TRY(cudaLaunchKernelEx(&cfg, kern, tq, td, b));
  if (st) {
    unsigned long long h[8];
    CUDA_TRY(cudaMemcpyAsync(h, st, sizeof(h), cudaMemcpyDeviceToHost, stream));
    CUDA_TRY(cudaStreamSynchronize(stream));
    cudaFree(st);
    const double pairs = kp.grid / 2.0, ep = 8.0 * kp.grid;
    fprintf(stderr, "[hiper pipe] maxsim%s: MMA thread %.0f cyc avg; waits acc %.1f%% full %.1f%%; "
            "epilogue drain %.0f cyc/tile, wait %.0f cyc/tile, tiles/warp %.0f\n",
            PACKED ? " (packed)" : "", h[2] / pairs, 100.0 * h[0] / h[2], 100.0 * h[1] / h[2],
            (double)h[3] / h[5], (double)h[4] / h[5], h[5] / ep);
  }
  CUDA_TRY(cudaGetLastError());
  TRY(profile_end(stream, ev));
  ++g_launches;
  return HIPER_OK;
}

// MODE 0 dense scores, 1 top-k (KR = ceil(k / 32) register ranks per lane), 2 scores + argmax;
// packed (a.recs) or dense; QW = kp.qw warps per query; H = kp.h MMA halves per chunk.
template <int MODE, int KR, bool PACKED>
static hiper_status launch_maxsim_qh(const KernelPlan& kp, const CUtensorMap& tq, const CUtensorMap& td,
                                     const MaxsimArgs& a, cudaStream_t stream) {
  if constexpr (PACKED) {
    if (kp.h != 1) return fail(HIPER_ERR_UNSUPPORTED, "packed tiles hold <= 256 rows");
    if (kp.qw == 1) return launch_maxsim_t<MODE, KR, true, 1, 1>(kp, tq, td, a, stream);
    if (kp.qw == 2) return launch_maxsim_t<MODE, KR, true, 2, 1>(kp, tq, td, a, stream);
    return launch_maxsim_t<MODE, KR, true, 4, 1>(kp, tq, td, a, stream);
  } else {
    if (kp.h == 1) {
      if (kp.qw == 1) return launch_maxsim_t<MODE, KR, false, 1, 1>(kp, tq, td, a, stream);
      if (kp.qw == 2) return launch_maxsim_t<MODE, KR, false, 2, 1>(kp, tq, td, a, stream);
      return launch_maxsim_t<MODE, KR, false, 4, 1>(kp, tq, td, a, stream);
    }
    if (kp.qw == 1) return launch_maxsim_t<MODE, KR, false, 1, 2>(kp, tq, td, a, stream);
    if (kp.qw == 2) return launch_maxsim_t<MODE, KR, false, 2, 2>(kp, tq, td, a, stream);
    return launch_maxsim_t<MODE, KR, false, 4, 2>(kp, tq, td, a, stream);
  }
}

static hiper_status launch_maxsim(int mode, int k, const KernelPlan& kp, const CUtensorMap& tq,
                                  const CUtensorMap& td, const MaxsimArgs& a, cudaStream_t stream) {
  if (kp.grid == 0) return HIPER_OK;
  if (mode == 2) {
    if (a.recs != nullptr || kp.qw != 1 || kp.h != 1)
      return fail(HIPER_ERR_UNSUPPORTED, "argmax capture needs a dense layout, q_max_len <= 32, d_max_len <= 256");
    return launch_maxsim_t<2, 1, false, 1, 1>(kp, tq, td, a, stream);
  }
  if (a.recs != nullptr) {  // packed corpus (N4)
    if (mode == 0) return launch_maxsim_qh<0, 1, true>(kp, tq, td, a, stream);
    if (k <= 32) return launch_maxsim_qh<1, 1, true>(kp, tq, td, a, stream);
    if (k <= 64) return launch_maxsim_qh<1, 2, true>(kp, tq, td, a, stream);
    return launch_maxsim_qh<1, 4, true>(kp, tq, td, a, stream);
  }
  if (mode == 0) return launch_maxsim_qh<0, 1, false>(kp, tq, td, a, stream);
  if (k <= 32) return launch_maxsim_qh<1, 1, false>(kp, tq, td, a, stream);
  if (k <= 64) return launch_maxsim_qh<1, 2, false>(kp, tq, td, a, stream);
  return launch_maxsim_qh<1, 4, false>(kp, tq, td, a, stream);
}

// list_len: keys per list (<= 128; 0 = k)
static hiper_status launch_merge(const uint64_t* lists, int32_t n_lists, int64_t list_stride,
                                 int32_t n_q, int64_t q_stride, int32_t k, uint64_t* out_keys,
                                 float* out_scores, int64_t* out_ids, cudaStream_t stream,
                                 int32_t list_len = 0) {
  if (n_q == 0) return HIPER_OK;
  const int threads = 256, qpb = threads / 32;
  const int blocks = (n_q + qpb - 1) / qpb;
  const int32_t ll = list_len > 0 ? list_len : k;
  // KR covers both the output k and the list length (a list is read KR x 32 keys at a time)
  const int32_t kr = std::max(k, ll);
  if (kr <= 32)
    topk_merge_kernel<1><<<blocks, threads, 0, stream>>>(lists, n_lists, list_stride, n_q, q_stride, k, out_keys, out_scores, out_ids, ll);
  else if (kr <= 64)
    topk_merge_kernel<2><<<blocks, threads, 0, stream>>>(lists, n_lists, list_stride, n_q, q_stride, k, out_keys, out_scores, out_ids, ll);
  else
    topk_merge_kernel<4><<<blocks, threads, 0, stream>>>(lists, n_lists, list_stride, n_q, q_stride, k, out_keys, out_scores, out_ids, ll);
  CUDA_TRY(cudaGetLastError());
  ++g_launches;
  return HIPER_OK;
}

// ============================================================================ communicator
struct hiper_comm_s {
  ncclComm_t comm = nullptr;
  int32_t world = 1, rank = 0, device = 0;
  // NEXT N2 peer windows (kernels/peer_gather.cuh): this rank's window [256 B ready word | 2 parity
  // buffers of win_bytes] exported with CUDA IPC; peer[r] = rank r's window mapped here (peer[rank] =
  // win).  Set up collectively on first use (peer_windows); epoch counts hiper_coltrast_loss calls.
  size_t win_bytes = 0;
  void* win = nullptr;
  std::vector<void*> peer;
  unsigned long long epoch = 0;
  bool ipc_failed = false;
};
static constexpr size_t kWinHeader = 256;

#define NCCL_TRY(expr)                                                                          \
  do {                                                                                          \
    ncclResult_t _r = (expr);                                                                   \
    if (_r != ncclSuccess)                                                                      \
      return fail(HIPER_ERR_NCCL, "%s: %s (%s:%d)", #expr, ncclGetErrorString(_r), __FILE__, __LINE__); \
  } while (0)

// A collective's enqueue can succeed while the communicator has already failed asynchronously (a
// peer died, a network error): ncclCommGetAsyncError is non-blocking and reports it.
static hiper_status nccl_async_check(const hiper_comm_s* c, const char* what) {
  ncclResult_t ar = ncclSuccess;
  NCCL_TRY(ncclCommGetAsyncError(c->comm, &ar));
  if (ar != ncclSuccess && ar != ncclInProgress)
    return fail(HIPER_ERR_NCCL, "%s: communicator async error: %s", what, ncclGetErrorString(ar));
  return HIPER_OK;
}

// a8: every rank's local [n_q][k] key list -> [world][n_q][k] on every rank (one ncclAllGather on
// `stream`, no host round trip), then the same deterministic merge + decode (a7/a9 kernel).
static hiper_status gather_merge(const hiper_comm_s* c, const uint64_t* local, uint64_t* gathered,
                                 int32_t n_q, int32_t k, float* out_scores, int64_t* out_ids,
                                 cudaStream_t stream);

extern "C" hiper_status hiper_shard_range(int64_t n, int32_t world, int32_t rank, int64_t* c0,
                                          int64_t* c1) {
  if (n < 0 || world < 1 || rank < 0 || rank >= world || !c0 || !c1)
    return fail(HIPER_ERR_INVALID_ARG, "bad shard arguments (n %lld, world %d, rank %d)", (long long)n,
                world, rank);
  // contiguous ranges, sizes differing by at most one: [rank * n / world, (rank + 1) * n / world)
  *c0 = (int64_t)((__int128)rank * n / world);
  *c1 = (int64_t)((__int128)(rank + 1) * n / world);
  return HIPER_OK;
}

extern "C" hiper_status hiper_comm_unique_id(uint8_t id[128]) {
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
  if (!id) return fail(HIPER_ERR_INVALID_ARG, "id is NULL");
  ncclUniqueId u;
  NCCL_TRY(ncclGetUniqueId(&u));
  memcpy(id, &u, 128);
  return HIPER_OK;
}

extern "C" hiper_status hiper_comm_create(const uint8_t id[128], int32_t world, int32_t rank,
                                          int32_t device, hiper_comm** out) {
  if (!id || !out) return fail(HIPER_ERR_INVALID_ARG, "NULL argument");
  if (world < 1 || rank < 0 || rank >= world) return fail(HIPER_ERR_INVALID_ARG, "bad world/rank");
  *out = nullptr;
  CUDA_TRY(cudaSetDevice(device));
  ncclUniqueId u;
  memcpy(&u, id, 128);
  hiper_comm_s* c = new hiper_comm_s();
  c->world = world;
  c->rank = rank;
  c->device = device;
  ncclResult_t r = ncclCommInitRank(&c->comm, world, u, rank);
  if (r != ncclSuccess) {
    delete c;
    return fail(HIPER_ERR_NCCL, "ncclCommInitRank: %s", ncclGetErrorString(r));
  }
  *out = c;
  return HIPER_OK;
}

static void release_windows(hiper_comm_s* c) {
  for (int32_t r = 0; r < (int32_t)c->peer.size(); ++r)
    if (r != c->rank && c->peer[r]) cudaIpcCloseMemHandle(c->peer[r]);
  if (c->win) cudaFree(c->win);
  c->peer.clear();
  c->win = nullptr;
  c->win_bytes = 0;
}

// Collective: every rank calls it with the same `bytes` (the same b, dp).  Allocates this rank's
// window, all-gathers the IPC handles over the communicator, maps every peer's window.
static hiper_status peer_windows(hiper_comm_s* c, size_t bytes, cudaStream_t stream) {
  if (c->win_bytes >= bytes && c->win) return HIPER_OK;
  CUDA_TRY(cudaStreamSynchronize(stream));
  release_windows(c);
  CUDA_TRY(cudaMalloc(&c->win, kWinHeader + 2 * bytes));
  CUDA_TRY(cudaMemset(c->win, 0, kWinHeader));  // ready epoch 0
  cudaIpcMemHandle_t h;
  CUDA_TRY(cudaIpcGetMemHandle(&h, c->win));
  static_assert(sizeof(cudaIpcMemHandle_t) == 64, "IPC handle size");
  uint8_t* dh = nullptr;
  CUDA_TRY(cudaMalloc(&dh, 64 * (size_t)(c->world + 2)));
  CUDA_TRY(cudaMemcpyAsync(dh, &h, 64, cudaMemcpyHostToDevice, stream));
  NCCL_TRY(ncclAllGather(dh, dh + 64, 64, ncclUint8, c->comm, stream));
  std::vector<cudaIpcMemHandle_t> all(c->world);
  CUDA_TRY(cudaMemcpyAsync(all.data(), dh + 64, 64 * (size_t)c->world, cudaMemcpyDeviceToHost, stream));
  CUDA_TRY(cudaStreamSynchronize(stream));
  TRY(nccl_async_check(c, "all-gather of IPC handles"));
  c->peer.assign(c->world, nullptr);
  for (int32_t r = 0; r < c->world; ++r) {
    if (r == c->rank) {
      c->peer[r] = c->win;
      continue;
    }
    if (cudaIpcOpenMemHandle(&c->peer[r], all[r], cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) {
      cudaGetLastError();
      c->peer[r] = nullptr;
      c->ipc_failed = true;  // e.g. ranks on different nodes: the NCCL gather remains
    }
  }
  // agree on success (every rank must take the same path) and make sure every rank has mapped every
  // window before any rank signals into one
  int32_t* flag = reinterpret_cast<int32_t*>(dh + 64 * (size_t)(c->world + 1));
  const int32_t bad = c->ipc_failed ? 1 : 0;
  CUDA_TRY(cudaMemcpyAsync(flag, &bad, 4, cudaMemcpyHostToDevice, stream));
  NCCL_TRY(ncclAllReduce(flag, flag, 1, ncclInt32, ncclSum, c->comm, stream));
  int32_t any_bad = 0;
  CUDA_TRY(cudaMemcpyAsync(&any_bad, flag, 4, cudaMemcpyDeviceToHost, stream));
  CUDA_TRY(cudaStreamSynchronize(stream));
  cudaFree(dh);
  if (any_bad) {
    c->ipc_failed = true;
    release_windows(c);
    return HIPER_OK;
  }
  c->win_bytes = bytes;
  c->epoch = 0;
  return HIPER_OK;
}

extern "C" hiper_status hiper_comm_destroy(hiper_comm* c) {
  if (!c) return HIPER_OK;
  release_windows(c);
  ncclResult_t r = c->comm ? ncclCommDestroy(c->comm) : ncclSuccess;
  delete c;
  if (r != ncclSuccess) return fail(HIPER_ERR_NCCL, "ncclCommDestroy: %s", ncclGetErrorString(r));
  return HIPER_OK;
}

extern "C" hiper_status hiper_comm_info(const hiper_comm* c, int32_t* world, int32_t* rank) {
  if (!c) return fail(HIPER_ERR_INVALID_ARG, "comm is NULL");
  if (world) *world = c->world;
  if (rank) *rank = c->rank;
  return HIPER_OK;
}

static hiper_status gather_merge(const hiper_comm_s* c, const uint64_t* local, uint64_t* gathered,
                                 int32_t n_q, int32_t k, float* out_scores, int64_t* out_ids,
                                 cudaStream_t stream) {
  NCCL_TRY(ncclAllGather(local, gathered, (size_t)n_q * k, ncclUint64, c->comm, stream));
  TRY(nccl_async_check(c, "ncclAllGather of top-k keys"));
  return launch_merge(gathered, c->world, (int64_t)n_q * k, n_q, k, k, nullptr, out_scores, out_ids,
                      stream);
}

extern "C" hiper_status hiper_topk_merge_keys(const uint64_t* lists, int32_t n_lists, int32_t n_q,
                                              int32_t k, float* out_scores, int64_t* out_ids,
                                              hiper_stream_t stream_) {
  g_launches = 0;
  HiperRange nv("hiper_topk_merge_keys");
  if (n_lists < 0 || n_q < 0) return fail(HIPER_ERR_INVALID_ARG, "n_lists / n_q < 0");
  if (k < 1) return fail(HIPER_ERR_INVALID_ARG, "k must be >= 1");
  if (k > kMaxK) return fail(HIPER_ERR_UNSUPPORTED, "k %d > %d", k, kMaxK);
  if (n_q == 0) return HIPER_OK;
  if (!out_scores || !out_ids || !is_device_ptr(out_scores) || !is_device_ptr(out_ids))
    return fail(HIPER_ERR_INVALID_ARG, "outputs must be device memory");
  if (n_lists > 0 && (!lists || !is_device_ptr(lists)))
    return fail(HIPER_ERR_INVALID_ARG, "lists must be device memory");
  return launch_merge(lists, n_lists, (int64_t)n_q * k, n_q, k, k, nullptr, out_scores, out_ids,
                      (cudaStream_t)stream_);
}

// ============================================================================ workspace layouts
struct TopkWs {
  size_t status = 0, progress = 0, qlens = 0, qlayout = 0, partial = 0, local = 0, gathered = 0,
         total = 0;
};
static constexpr int32_t kLockstepWindow = 192;  // chunks (12 MB of a 256 x 128 bf16 corpus)

// n_q_pad / n_parts: the kernel plan's (they depend on the query slot size)
static void topk_ws_layout(int32_t n_q, int32_t dim, int32_t n_q_pad, int32_t n_parts, int32_t k,
                           int32_t world, bool with_comm, TopkWs& w) {
  size_t off = 0;
  w.status = off;
  off += 256;
  w.progress = off;
  off += 1024;  // up to 256 pairs
  w.qlens = off;
  off = align_up(off + (size_t)std::max(n_q, 1) * 4, 1024);
  w.qlayout = off;
  off = align_up(off + q_layout_bytes_max(n_q, dim), 1024);
  w.partial = off;
  off = align_up(off + (size_t)n_parts * kEpiGroups * n_q_pad * k * 8, 256);
  w.local = off;
  if (with_comm) off = align_up(off + (size_t)std::max(n_q, 1) * k * 8, 256);
  w.gathered = off;
  if (with_comm) off = align_up(off + (size_t)world * std::max(n_q, 1) * k * 8, 256);
  w.total = off;
}

// Kernel slots of an index: chunks, or the tiles of a packed index (N4).
static int64_t index_slots(const hiper_index* ix) { return ix->packed ? ix->n_tiles : ix->n; }
static int32_t index_slot_rows(const hiper_index* ix) { return ix->packed ? kTileRows : ix->ld_pad; }
static void set_packed_args(const hiper_index* ix, MaxsimArgs& a) {
  if (!ix->packed) return;
  a.recs = ix->recs;
}

static hiper_status check_ws(const void* ws, size_t have, size_t need) {
  if (!ws) return fail(HIPER_ERR_WORKSPACE, "workspace is NULL (need %zu bytes)", need);
  if (((uintptr_t)ws & 1023) != 0) return fail(HIPER_ERR_WORKSPACE, "workspace must be 1024-B aligned");
  if (have < need) return fail(HIPER_ERR_WORKSPACE, "workspace too small: %zu < %zu", have, need);
  return HIPER_OK;
}

static size_t pooled_ws_size(const hiper_index* ix, int32_t n_q, int32_t k, const hiper_comm* comm,
                             bool topk);

extern "C" size_t hiper_maxsim_topk_workspace_size(const hiper_index* ix, int32_t n_q, int32_t k,
                                                   const hiper_comm* comm) {
  if (!ix || n_q < 0 || k < 1) return 0;
  if (ix->pooled) return pooled_ws_size(ix, n_q, k, comm, true);
  int num_sms = 148;
  if (cudaDeviceGetAttribute(&num_sms, cudaDevAttrMultiProcessorCount, ix->device) != cudaSuccess) {
    cudaGetLastError();
    num_sms = 148;
  }
  // the largest layout over the query slot sizes (this entry point does not take q_max_len)
  size_t total = 0;
  for (int32_t qs = 32; qs <= 128; qs *= 2) {
    const int32_t nqp = n_q_pad_of(n_q, qs);
    TopkWs w;
    topk_ws_layout(n_q, ix->dim, nqp,
                   choose_parts_topk(nqp * qs / 256, index_slots(ix), num_sms / 2,
                                     (int64_t)index_slot_rows(ix) * ix->dim * 2, nqp, k),
                   k, comm ? comm->world : 1, comm != nullptr, w);
    total = std::max(total, w.total);
  }
  return total;
}

extern "C" hiper_status hiper_workspace_status(const void* workspace, hiper_stream_t stream) {
  if (!workspace) return fail(HIPER_ERR_WORKSPACE, "workspace is NULL");
  return sync_status((const uint32_t*)workspace, (cudaStream_t)stream);
}

// ============================================================================ top-k search
// ============================================================================ pooled limit case (a12)
// One vector per query and per chunk: S = <NORM(q), NORM(c)> via the K-pipelined pair GEMM with a
// fused per-query register top-k (kernels/pooled_sm100_pair.cuh).
constexpr int kPooledKP = 16;  // register top-k slots per query thread (k <= 16; larger k: warp lists)
constexpr int kPooledKP8 = 8;  // the short register list (k <= 8)

struct PooledPlan {
  int32_t n_qtiles = 0, n_ctiles = 0, n_parts = 0, n_stages = 0, q_pad = 0;
  uint32_t stage_bytes = 32768u, smem_bytes = 0;
  int grid = 0, cl = 2;
};

// Pooled top-k cluster shape: 4 = two CTA pairs sharing each chunk tile through TMA multicast
// (HIPER_POOLED_MC=1), 2 = one pair per cluster.
static int pooled_cluster(bool topk) {
  static const int cl = [] {
    const char* e = getenv("HIPER_POOLED_MC");
    return (e && e[0] == '1') ? 4 : 2;
  }();
  return topk ? cl : 2;
}
static int32_t pooled_qtiles(int32_t n_q, int cl) {
  const int32_t qt = (int32_t)((std::max(n_q, 1) + 255) / 256);
  return cl == 4 ? (qt + 1) / 2 * 2 : qt;
}

static hiper_status plan_pooled(const DevInfo& di, int32_t n_q, int64_t n_chunks, PooledPlan& pp,
                                bool topk = true, int32_t k = 1, bool append = false) {
  pp.cl = pooled_cluster(topk);
  pp.n_qtiles = pooled_qtiles(n_q, pp.cl);
  pp.q_pad = pp.n_qtiles * 256;
  const int64_t ct = (n_chunks + 255) / 256;
  if (ct > 0x7FFFFFFF) return fail(HIPER_ERR_UNSUPPORTED, "too many chunks");
  pp.n_ctiles = (int32_t)ct;
  int pairs = di.num_sms / 2;
  // ablation only: fewer resident pairs (the per-SM vs chip-wide L2->SMEM throughput experiment);
  // must keep choose_parts() equal to the workspace sizing (it does for divisors of num_sms / 2)
  if (const char* e = getenv("HIPER_POOLED_PAIRS")) pairs = std::max(1, std::min(pairs, atoi(e)));
  pp.n_parts = choose_parts(pp.n_qtiles / (pp.cl / 2), pp.n_ctiles, di.num_sms / pp.cl);
  uint32_t fixed = 1024u + 1024u;  // align slack, barriers
  if (topk && k > kPooledKP && !append) fixed += 128u * (uint32_t)(k | 1) * 8u + 512u + 8192u;  // heaps, locks, top-8
  pp.n_stages = (int32_t)std::min<uint32_t>(8u, ((uint32_t)di.max_smem - fixed) / pp.stage_bytes);
  if (pp.n_stages < 2) return fail(HIPER_ERR_UNSUPPORTED, "not enough shared memory");
  pp.smem_bytes = fixed + pp.n_stages * pp.stage_bytes;
  pp.grid = (int)std::min<int64_t>((int64_t)(pp.n_qtiles / (pp.cl / 2)) * pp.n_parts,
                                   pairs / (pp.cl / 2)) * pp.cl;
  return HIPER_OK;
}

template <int MODE>
static hiper_status launch_pooled(const PooledPlan& pp, const CUtensorMap& tq, const CUtensorMap& tc,
                                  const PooledArgs& a, cudaStream_t stream) {
  if (pp.grid == 0 || pp.n_parts == 0) return HIPER_OK;
  static const bool pstats_on = getenv("HIPER_PIPE_STATS") != nullptr;
  auto kern = pp.cl == 4 ? pooled_sm100_pair_kernel<MODE, kPooledKP, 0, 4>
              : pstats_on ? pooled_sm100_pair_kernel<MODE, kPooledKP, 0, 2, true>
                          : pooled_sm100_pair_kernel<MODE, kPooledKP, 0>;
  // k <= 8 (and the APPEND sample pre-pass): an 8-slot register list, half the work per insertion
  if constexpr (MODE == 1) {
    static const bool kp8_off = getenv("HIPER_POOLED_KP8") && getenv("HIPER_POOLED_KP8")[0] == '0';  // A/B
    if (pp.cl == 2 && a.k <= kPooledKP8 && !kp8_off)
      kern = pstats_on ? pooled_sm100_pair_kernel<MODE, kPooledKP8, 0, 2, true>
                       : pooled_sm100_pair_kernel<MODE, kPooledKP8, 0>;
  }
  if (MODE == 1 && a.k > kPooledKP) {  // shared-memory heaps, or the APPEND candidate buffers
    if (pp.cl != 2) return fail(HIPER_ERR_UNSUPPORTED, "pooled k > %d with HIPER_POOLED_MC", kPooledKP);
    if (a.cand != nullptr)
      kern = pstats_on ? pooled_sm100_pair_kernel<MODE, -1, 0, 2, true> : pooled_sm100_pair_kernel<MODE, -1, 0, 2>;
    else
      kern = pstats_on ? pooled_sm100_pair_kernel<MODE, 0, 0, 2, true> : pooled_sm100_pair_kernel<MODE, 0, 0, 2>;
  }
  if (MODE == 1 && debug_mode() == 1) kern = pooled_sm100_pair_kernel<MODE, kPooledKP, 1, 2, true>;
  if (MODE == 1 && debug_mode() == 2) kern = pooled_sm100_pair_kernel<MODE, kPooledKP, 2, 2, true>;
  if (MODE == 1 && debug_mode() == 3) kern = pooled_sm100_pair_kernel<MODE, kPooledKP, 3, 2, true>;
  if (MODE == 1 && debug_mode() == 4) kern = pooled_sm100_pair_kernel<MODE, kPooledKP, 4, 2, true>;
  CUDA_TRY(set_max_smem((const void*)kern, (int)pp.smem_bytes));
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)pp.grid);
  cfg.blockDim = dim3(kMaxsimThreads);
  cfg.dynamicSmemBytes = pp.smem_bytes;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = (unsigned)pp.cl;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  ProfTicket ev;
  // diagnostics only (HIPER_PIPE_STATS=1): pipeline wait/drain cycle counters, printed to stderr
  static const bool stats_on = getenv("HIPER_PIPE_STATS") != nullptr;
  unsigned long long* st = nullptr;
  PooledArgs b = a;
  if (stats_on) {
    CUDA_TRY(cudaMalloc(&st, 16 * sizeof(unsigned long long)));
    CUDA_TRY(cudaMemsetAsync(st, 0, 16 * sizeof(unsigned long long), stream));
    b.stats = st;
  }
  TRY(profile_begin(stream, HIPER_PROF_POOLED, &ev));
  CUDA_TRY(cudaLaunchKernelEx(&cfg, kern, tq, tc, b));
  TRY(profile_end(stream, ev));
  ++g_launches;
  if (st) {
    unsigned long long h[16];
    CUDA_TRY(cudaMemcpyAsync(h, st, sizeof(h), cudaMemcpyDeviceToHost, stream));
    CUDA_TRY(cudaStreamSynchronize(stream));
    cudaFree(st);
    const double pairs = pp.grid / 2.0, ep = 8.0 * pp.grid;  // MMA threads, epilogue warps
    fprintf(stderr, "[hiper pipe] pooled: MMA thread %.0f cyc avg; waits acc %.1f%% full %.1f%%; "
            "epilogue drain %.0f cyc/tile, wait %.0f cyc/tile, tiles/warp %.0f; per thread-tile: "
            "blocks past the threshold %.3f, inserts %.3f; shared-list sections %llu (%.0f cyc spin, "
            "%.0f cyc held avg)\n",
            h[2] / pairs, 100.0 * h[0] / h[2], 100.0 * h[1] / h[2], (double)h[3] / h[5],
            (double)h[4] / h[5], h[5] / ep, (double)h[6] / (32.0 * h[5]), (double)h[7] / (32.0 * h[5]),
            h[8], (double)h[9] / std::max(1ull, h[8]), (double)h[10] / std::max(1ull, h[8]));
  }
  return HIPER_OK;
}

// a12 with the chunk tile stationary (kernels/pooled_cs_sm100.cuh): every pair owns a contiguous
// range of chunk tiles and streams all query tiles against each.  Exact and tested, but measured
// slower than the streaming kernel at config 5 (0.78 vs 0.81 of burst, same box: the query feed from
// L2 with <= 3 stages beside the resident tile; profiles/r02/ablation/pooled_cs.txt), so it is
// opt-in: HIPER_POOLED_CS=2 uses it for the register top-k (k <= kPooledKP) when the resident tile
// leaves >= 2 query stages and every pair gets >= 2 chunk tiles, =1 forces it on any corpus (tests:
// min(pairs, chunk tiles) pairs).  HIPER_POOLED_CS_N = chunk tile width (default 224, the best
// measured), HIPER_POOLED_CS_A = query stage width 32 | 64 (default 64).
struct PooledCsPlan {
  bool use = false;
  int32_t n_parts = 0, n_stages = 0, two_slots = 0, tile_n = 256, n_ctiles = 0, a_cols = 32;
  uint32_t smem_bytes = 0;
  int grid = 0;
};
static void plan_pooled_cs(int num_sms, int max_smem, int32_t n_q, int64_t n_chunks, int32_t dim,
                           int32_t k, bool topk, PooledCsPlan& cp) {
  cp = PooledCsPlan{};
  const char* e = getenv("HIPER_POOLED_CS");
  const int mode = e ? atoi(e) : 0;  // 0 off, 1 forced, 2 auto
  if (mode == 0 || !topk || k > kPooledKP || pooled_cluster(true) != 2 || n_chunks <= 0) return;
  const int64_t nkb = num_kb_of(dim);
  const char* en = getenv("HIPER_POOLED_CS_N");
  const int64_t tn = en ? std::max(16, std::min(256, atoi(en) / 16 * 16)) : 224;
  const char* ea = getenv("HIPER_POOLED_CS_A");
  const int64_t ac = (ea && atoi(ea) == 32) ? 32 : 64;
  const int64_t fixed = 1024 + 1024;  // align slack, barriers + TMEM pointer
  const int64_t avail = (int64_t)max_smem - fixed - nkb * tn * 64;
  const int64_t S = std::min<int64_t>(12, avail / (256 * ac));
  const int32_t pairs = num_sms / 2;
  const int64_t ct = (n_chunks + tn - 1) / tn;
  if (S < (ac == 64 ? 2 : 3) || (mode == 2 && ct < 2 * (int64_t)pairs)) return;
  const int32_t nqt = (int32_t)((std::max(n_q, 1) + 255) / 256);
  cp.use = true;
  cp.n_parts = (int32_t)std::min<int64_t>(pairs, ct);
  cp.n_stages = (int32_t)S;
  cp.two_slots = (nqt & 1) ? 1 : 0;
  cp.tile_n = (int32_t)tn;
  cp.a_cols = (int32_t)ac;
  cp.n_ctiles = (int32_t)ct;
  cp.smem_bytes = (uint32_t)(fixed + nkb * tn * 64 + S * 256 * ac);
  cp.grid = 2 * cp.n_parts;
}

static hiper_status launch_pooled_cs(const PooledCsPlan& cp, const CUtensorMap& tq32,
                                     const CUtensorMap& tc, const PooledCsArgs& a, cudaStream_t stream) {
  static const bool stats_on = getenv("HIPER_PIPE_STATS") != nullptr;
  auto kern = cp.a_cols == 64
                  ? (stats_on ? pooled_cs_sm100_kernel<kPooledKP, 64, true> : pooled_cs_sm100_kernel<kPooledKP, 64>)
                  : (stats_on ? pooled_cs_sm100_kernel<kPooledKP, 32, true> : pooled_cs_sm100_kernel<kPooledKP, 32>);
  CUDA_TRY(set_max_smem((const void*)kern, (int)cp.smem_bytes));
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)cp.grid);
  cfg.blockDim = dim3(kMaxsimThreads);
  cfg.dynamicSmemBytes = cp.smem_bytes;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  unsigned long long* st = nullptr;
  PooledCsArgs b = a;
  if (stats_on) {
    CUDA_TRY(cudaMalloc(&st, 16 * sizeof(unsigned long long)));
    CUDA_TRY(cudaMemsetAsync(st, 0, 16 * sizeof(unsigned long long), stream));
    b.stats = st;
  }
  ProfTicket ev;
  TRY(profile_begin(stream, HIPER_PROF_POOLED, &ev));
  CUDA_TRY(cudaLaunchKernelEx(&cfg, kern, tq32, tc, b));
  TRY(profile_end(stream, ev));
  ++g_launches;
  if (st) {
    unsigned long long h[16];
    CUDA_TRY(cudaMemcpyAsync(h, st, sizeof(h), cudaMemcpyDeviceToHost, stream));
    CUDA_TRY(cudaStreamSynchronize(stream));
    cudaFree(st);
    const double pairs = cp.grid / 2.0, ep = 8.0 * cp.grid;
    fprintf(stderr, "[hiper pipe] pooled_cs: MMA thread %.0f cyc avg; waits acc %.1f%% A %.1f%% B %.1f%%; "
            "epilogue drain %.0f cyc/tile, wait %.0f cyc/tile, tiles/warp %.0f; per thread-tile: "
            "blocks past the threshold %.3f, list loads %.3f\n",
            h[2] / pairs, 100.0 * h[0] / h[2], 100.0 * h[1] / h[2], 100.0 * h[6] / h[2],
            (double)h[3] / h[5], (double)h[4] / h[5], h[5] / ep, (double)h[7] / (32.0 * h[5]),
            (double)h[8] / (32.0 * h[5]));
  }
  return HIPER_OK;
}

struct PooledWs {
  size_t status = 0, progress = 0, qlens = 0, qlayout = 0, partial = 0, local = 0, gathered = 0,
         gthr = 0, pub8 = 0, thrk = 0, cand = 0, ccnt = 0, total = 0;
};
// Pooled top-k with 16 < k <= 128, APPEND path: a pre-pass takes the exact top-k of a corpus sample
// (the first S chunks, whole 256-chunk tiles, S ~ n / 32 and >= 8k) with the heap kernel; the k-th
// key of the sample, T_q, bounds the k-th key of the corpus from below, so the main pass only has to
// append the keys >= T_q (~32 k per query) and a warp per query selects the top k of them.  The
// heaps leave shared memory to the pipeline (6 stages instead of 3).  0 = no APPEND (small corpora,
// or HIPER_POOLED_APPEND=0).
static int64_t pooled_append_sample(int64_t n_chunks, int32_t k) {
  static const bool off = getenv("HIPER_POOLED_APPEND") && getenv("HIPER_POOLED_APPEND")[0] == '0';
  if (off || k <= kPooledKP) return 0;
  static const int64_t div = getenv("HIPER_POOLED_SAMPLE_DIV") ? atoll(getenv("HIPER_POOLED_SAMPLE_DIV")) : 32;
  int64_t s = std::max<int64_t>(n_chunks / std::max<int64_t>(div, 4), 8 * (int64_t)k);
  s = (s + 255) / 256 * 256;
  return s * 4 <= n_chunks ? s : 0;
}
// candidate slots per (query, partition, group) segment: 3x the expected k * div / (2P) + 16
// (HIPER_POOLED_APPEND_CAP: tests of the overflow fallback)
static int32_t pooled_append_cap(int32_t k, int32_t n_parts) {
  if (const char* e = getenv("HIPER_POOLED_APPEND_CAP")) return std::max(1, atoi(e));
  static const int64_t div = getenv("HIPER_POOLED_SAMPLE_DIV") ? atoll(getenv("HIPER_POOLED_SAMPLE_DIV")) : 32;
  const int64_t e = (int64_t)k * std::max<int64_t>(div, 4) / (2 * std::max(n_parts, 1));
  return (int32_t)std::max<int64_t>(32, (3 * e + 16 + 7) / 8 * 8);
}
static void pooled_ws_layout(int32_t n_q, int32_t dim, int32_t n_parts, int32_t q_pad, int32_t k,
                             int32_t world, bool with_comm, PooledWs& w, bool append = false) {
  size_t off = 0;
  w.status = off;
  off += 256;
  w.progress = off;
  off += 1024;
  w.qlens = off;
  off = align_up(off + (size_t)std::max(n_q, 1) * 4, 1024);
  w.qlayout = off;
  off = align_up(off + (size_t)std::max(n_q, 1) * dim * 2, 1024);
  w.partial = off;
  off = align_up(off + (size_t)n_parts * kEpiGroups * q_pad * k * 8, 256);
  w.local = off;
  if (with_comm) off = align_up(off + (size_t)std::max(n_q, 1) * k * 8, 256);
  w.gathered = off;
  if (with_comm) off = align_up(off + (size_t)world * std::max(n_q, 1) * k * 8, 256);
  w.gthr = off;
  off = align_up(off + (size_t)q_pad * 8, 256);
  w.pub8 = off;  // k > kPooledKP: [q_pad][n_parts] published 8th-best keys
  if (k > kPooledKP) off = align_up(off + (size_t)q_pad * std::max(n_parts, 1) * 8, 256);
  w.thrk = off;  // APPEND: [n_q][k] the sample's top-k keys (T_q = the last)
  w.cand = off;
  w.ccnt = off;
  if (append) {
    off = align_up(off + (size_t)std::max(n_q, 1) * k * 8, 256);
    const size_t segs = (size_t)std::max(n_q, 1) * std::max(n_parts, 1) * kEpiGroups;
    w.cand = off;  // [n_q][P][2][cap] candidate keys, one segment per unit thread
    off = align_up(off + segs * pooled_append_cap(k, n_parts) * 8, 256);
    w.ccnt = off;  // [n_q][P][2] segment counts
    off = align_up(off + segs * 4, 256);
  }
  w.total = off;
}

static hiper_status pooled_search(const hiper_index* ix, const void* q_tokens, hiper_dtype dtype,
                                  const int32_t* q_lens, int32_t n_q, int32_t dim, int32_t k,
                                  uint32_t flags, const hiper_comm* comm, void* workspace,
                                  size_t workspace_bytes, float* out_scores, int64_t* out_ids,
                                  float* dense_scores, cudaStream_t stream,
                                  uint64_t* out_keys = nullptr, bool allow_append = true) {
  DevInfo di;
  TRY(device_info(di));
  PooledPlan pp;
  TRY(plan_pooled(di, n_q, ix->n, pp, dense_scores == nullptr, k));
  PooledCsPlan cp;
  plan_pooled_cs(di.num_sms, di.max_smem, n_q, ix->n, dim, k, dense_scores == nullptr, cp);
  const int32_t world = comm ? comm->world : 1;
  const bool glists = !dense_scores && k > kPooledKP;  // one shared list per query (see the kernel)
  const bool append_ws = glists && pp.cl == 2 && pooled_append_sample(ix->n, k) > 0;
  const int64_t sample = allow_append && append_ws ? pooled_append_sample(ix->n, k) : 0;
  PooledWs w;
  pooled_ws_layout(n_q, dim, std::max(pp.n_parts, cp.n_parts), pp.q_pad, dense_scores ? 1 : k, world,
                   comm != nullptr, w, append_ws);
  TRY(check_ws(workspace, workspace_bytes, w.total));
  uint8_t* ws = (uint8_t*)workspace;
  uint32_t* status = (uint32_t*)(ws + w.status);
  int32_t* qlens_dev = (int32_t*)(ws + w.qlens);
  __nv_bfloat16* qlayout = (__nv_bfloat16*)(ws + w.qlayout);
  uint64_t* partial = (uint64_t*)(ws + w.partial);
  CUDA_TRY(cudaMemsetAsync(status, 0, sizeof(uint32_t), stream));
  CUDA_TRY(cudaMemsetAsync(ws + w.progress, 0xFF, w.qlens - w.progress, stream));  // "not started"
  TRY(stage_h2d(qlens_dev, q_lens, (size_t)n_q * 4, stream));
  TRY(launch_norm(q_tokens, dtype, n_q, 1, qlens_dev, n_q, 1, dim, flags, qlayout, status, stream));
  if (flags & HIPER_VALIDATE_SYNC) TRY(sync_status(status, stream));
  PooledArgs a{};
  a.n_q = n_q;
  a.n_qtiles = pp.n_qtiles;
  a.n_ctiles = pp.n_ctiles;
  a.n_parts = pp.n_parts;
  a.num_kb = num_kb_of(dim);
  a.k = dense_scores ? 1 : k;
  a.n_stages = pp.n_stages;
  a.stage_bytes = pp.stage_bytes;
  a.q_pad = pp.q_pad;
  a.n_chunks = ix->n;
  a.id_base = ix->id_base;
  a.partial = partial;
  a.scores = dense_scores;
  a.score_ld = ix->n;
  // The L2 lockstep pays off for the token MaxSim kernel under the power cap (less DRAM, higher
  // clocks), not here: the pooled kernel's feed is latency-bound, and without it config 5 runs 2.6%
  // faster in a burst and 1% faster sustained (profiles/r02/ablation/pooled_lockstep.txt).
  // HIPER_POOLED_LOCKSTEP=1 turns it on.
  a.progress = (getenv("HIPER_POOLED_LOCKSTEP") && getenv("HIPER_POOLED_LOCKSTEP")[0] == '1')
                   ? (uint32_t*)(ws + w.progress) : nullptr;
  a.window = 16;
  if (const char* e = getenv("HIPER_POOLED_WINDOW")) a.window = std::max(1, atoi(e));  // ablation
  if (!dense_scores && getenv("HIPER_NO_SHARED_BOUND") == nullptr) {
    a.gthr = (unsigned long long*)(ws + w.gthr);
    CUDA_TRY(cudaMemsetAsync(a.gthr, 0, (size_t)pp.q_pad * 8, stream));
    if (glists && getenv("HIPER_NO_PUB8") == nullptr) {
      a.pub8 = (unsigned long long*)(ws + w.pub8);
      CUDA_TRY(cudaMemsetAsync(a.pub8, 0, (size_t)pp.q_pad * std::max(pp.n_parts, 1) * 8, stream));
    }
  }
  if (sample > 0) {
    // APPEND: (1) the sample with the fast register kernel (per-(partition, group) top-16 lists, no
    // shared pruning bound, so each list is its own sub-sample's exact top 16) -> T_q = the k-th key of
    // the union of the lists: a k-th largest of real corpus keys, so at least k corpus keys are >= T_q;
    // and as close to the sample's own k-th as long as no list holds more than 16 of its top k
    alignas(64) CUtensorMap tq;
    TRY(make_tmap(&tq, qlayout, n_q, dim, 128));
    PooledPlan p0;
    TRY(plan_pooled(di, n_q, sample, p0, true, kPooledKP));
    // each (partition, group) list keeps its sub-sample's top kp0: any k-th largest key of the union
    // of real keys is a valid bound once the union holds >= k keys (2 P kp0 >= k), and it equals the
    // sample's own k-th unless one list holds more than kp0 of the sample's top k (expected k / 2P
    // per list).  A short list pays ~kp0 (1 + ln(n / kp0)) insertions instead of 16 (1 + ln(n / 16)).
    const int32_t per = (k + 2 * p0.n_parts - 1) / std::max(1, 2 * p0.n_parts);
    int32_t kp0 = std::min(kPooledKP, std::max(4, 3 * per));
    if (const char* e = getenv("HIPER_PREPASS_KP")) kp0 = std::min(kPooledKP, std::max(per, atoi(e)));  // A/B
    PooledArgs a0 = a;
    a0.k = kp0;
    a0.n_ctiles = p0.n_ctiles;
    a0.n_parts = p0.n_parts;
    a0.n_stages = p0.n_stages;
    a0.n_chunks = sample;
    a0.gthr = nullptr;
    a0.pub8 = nullptr;
    TRY(launch_pooled<1>(p0, tq, ix->tmap, a0, stream));
    uint64_t* thrk = (uint64_t*)(ws + w.thrk);
    TRY(launch_merge(partial, p0.n_parts * kEpiGroups, (int64_t)p0.q_pad * kp0, n_q, kp0, k,
                     thrk, nullptr, nullptr, stream, kp0));
    // (2) the whole corpus: every key >= T_q into the query's candidate buffer
    PooledPlan p1;
    TRY(plan_pooled(di, n_q, ix->n, p1, true, k, /*append=*/true));
    PooledArgs a1 = a;
    a1.n_stages = p1.n_stages;
    a1.n_parts = p1.n_parts;
    a1.gthr = nullptr;
    a1.pub8 = nullptr;
    if (p1.n_parts != pp.n_parts) return fail(HIPER_ERR_UNSUPPORTED, "APPEND partition plan mismatch");
    const int32_t cap = pooled_append_cap(k, p1.n_parts);
    uint32_t* ccnt = (uint32_t*)(ws + w.ccnt);
    a1.cand = (uint64_t*)(ws + w.cand);
    a1.cand_cnt = ccnt;  // every (q < n_q, p, g) count is written by its unit thread
    a1.cand_cap = cap;
    a1.cand_thr = thrk + (k - 1);
    a1.thr_stride = k;
    if (a1.progress != nullptr)
      CUDA_TRY(cudaMemsetAsync(ws + w.progress, 0xFF, w.qlens - w.progress, stream));  // "not started"
    TRY(launch_pooled<1>(p1, tq, ix->tmap, a1, stream));
    // (3) a warp per query: the top k of its buffer, as keys or decoded (this shard's, or the global
    // answer after the all-gather)
    uint64_t* local = (uint64_t*)(ws + w.local);
    uint64_t* keys_to = out_keys ? out_keys : ((comm && comm->world > 1) ? local : nullptr);
    const int blocks = (n_q + 7) / 8;
#define HIPER_SELECT(KR)                                                                          \
  cand_select_kernel<KR><<<blocks, 256, 0, stream>>>(a1.cand, ccnt, p1.n_parts * kEpiGroups, cap, \
                                                     n_q, k, keys_to,                              \
                                                     keys_to ? nullptr : out_scores,              \
                                                     keys_to ? nullptr : out_ids, status)
    if (k <= 32) HIPER_SELECT(1); else if (k <= 64) HIPER_SELECT(2); else HIPER_SELECT(4);
#undef HIPER_SELECT
    CUDA_TRY(cudaGetLastError());
    ++g_launches;
    // a buffer that overflowed (the sample was unrepresentative) cannot be trusted: redo the batch on
    // the heap path (one host sync per call on this path)
    uint32_t h = 0;
    CUDA_TRY(cudaMemcpyAsync(&h, status, sizeof(h), cudaMemcpyDeviceToHost, stream));
    CUDA_TRY(cudaStreamSynchronize(stream));
    if (h & 16u)
      return pooled_search(ix, q_tokens, dtype, q_lens, n_q, dim, k, flags, comm, workspace,
                           workspace_bytes, out_scores, out_ids, dense_scores, stream, out_keys, false);
    if (out_keys || !comm || comm->world == 1) return HIPER_OK;
    return gather_merge(comm, local, (uint64_t*)(ws + w.gathered), n_q, k, out_scores, out_ids, stream);
  }
  if (ix->n > 0) {
    alignas(64) CUtensorMap tq;
    TRY(make_tmap(&tq, qlayout, n_q, dim, 128));
    if (dense_scores) return launch_pooled<0>(pp, tq, ix->tmap, a, stream);
    if (cp.use) {
      alignas(64) CUtensorMap tq32, tcn;
      TRY(make_tmap(&tq32, qlayout, n_q, dim, 128, cp.a_cols));
      TRY(make_tmap(&tcn, ix->tok, ix->n, dim, cp.tile_n / 2));
      PooledCsArgs c{};
      c.n_q = n_q;
      c.n_qtiles = pp.n_qtiles;
      c.n_ctiles = cp.n_ctiles;
      c.tile_n = cp.tile_n;
      c.a_cols = cp.a_cols;
      c.dbg = getenv("HIPER_POOLED_CS_DBG") ? atoi(getenv("HIPER_POOLED_CS_DBG")) : 0;
      c.n_parts = cp.n_parts;
      c.num_kb = num_kb_of(dim);
      c.k = k;
      c.n_stages = cp.n_stages;
      c.q_pad = pp.q_pad;
      c.two_slots = cp.two_slots;
      c.n_chunks = ix->n;
      c.id_base = ix->id_base;
      c.partial = partial;
      c.gthr = a.gthr;
      TRY(launch_pooled_cs(cp, tq32, tcn, c, stream));
    } else if (pp.cl == 4) {  // chunk halves of 64 rows, multicast to both pairs of a cluster
      alignas(64) CUtensorMap tc64;
      TRY(make_tmap(&tc64, ix->tok, ix->n, dim, 64));
      TRY(launch_pooled<1>(pp, tq, tc64, a, stream));
    } else {
      TRY(launch_pooled<1>(pp, tq, ix->tmap, a, stream));
    }
  }
  // the per-(partition, group) lists; k > kPooledKP: one (shared-heap) list per partition, in the
  // group-0 slot of each partition
  // chunk-stationary kernel: lists [pair][slot] (slot 0 only when the query tiles are even)
  const bool one_slot = glists || (cp.use && !cp.two_slots);
  const int32_t n_lists =
      ix->n > 0 ? (cp.use ? cp.n_parts : pp.n_parts) * (one_slot ? 1 : kEpiGroups) : 0;
  const int64_t list_stride = (int64_t)pp.q_pad * k * (one_slot ? kEpiGroups : 1);
  if (out_keys)  // this shard's top-k keys (a8's all-gather payload)
    return launch_merge(partial, n_lists, list_stride, n_q, k, k, out_keys, nullptr, nullptr, stream);
  if (!comm || comm->world == 1)
    return launch_merge(partial, n_lists, list_stride, n_q, k, k, nullptr, out_scores, out_ids, stream);
  uint64_t* local = (uint64_t*)(ws + w.local);
  uint64_t* gathered = (uint64_t*)(ws + w.gathered);
  TRY(launch_merge(partial, n_lists, list_stride, n_q, k, k, local, nullptr, nullptr, stream));
  return gather_merge(comm, local, gathered, n_q, k, out_scores, out_ids, stream);
}

static size_t pooled_ws_size(const hiper_index* ix, int32_t n_q, int32_t k, const hiper_comm* comm,
                             bool topk) {
  int num_sms = 148;
  if (cudaDeviceGetAttribute(&num_sms, cudaDevAttrMultiProcessorCount, ix->device) != cudaSuccess) {
    cudaGetLastError();
    num_sms = 148;
  }
  const int cl = pooled_cluster(topk);
  const int32_t qt = pooled_qtiles(n_q, cl);
  const int32_t ct = (int32_t)((ix->n + 255) / 256);
  int max_smem = 0;
  if (cudaDeviceGetAttribute(&max_smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, ix->device) != cudaSuccess) {
    cudaGetLastError();
    max_smem = 232448;
  }
  PooledCsPlan cp;
  plan_pooled_cs(num_sms, max_smem, n_q, ix->n, ix->dim, k, topk, cp);
  PooledWs w;
  pooled_ws_layout(n_q, ix->dim, std::max(choose_parts(qt / (cl / 2), ct, num_sms / cl), cp.n_parts), qt * 256, k,
                   comm ? comm->world : 1, comm != nullptr, w,
                   topk && cl == 2 && pooled_append_sample(ix->n, k) > 0);
  return w.total;
}

// Steps a2-a9.  out_keys != NULL (comm == NULL): stop after the intra-GPU merge and write this shard's
// top-k as sortable keys (a8's all-gather payload, hiper_maxsim_topk_keys) instead of decoding.
static hiper_status topk_search(const hiper_index* ix, const void* q_tokens, hiper_dtype dtype,
                                const int32_t* q_lens, int32_t n_q, int32_t q_max_len, int32_t dim,
                                int32_t k, uint32_t flags, const hiper_comm* comm, void* workspace,
                                size_t workspace_bytes, float* out_scores, int64_t* out_ids,
                                uint64_t* out_keys, cudaStream_t stream) {
  if (!ix) return fail(HIPER_ERR_INVALID_ARG, "index is NULL");
  if (dim != ix->dim) return fail(HIPER_ERR_DIM_MISMATCH, "query dim %d != index dim %d", dim, ix->dim);
  if (k < 1) return fail(HIPER_ERR_INVALID_ARG, "k must be >= 1");
  if (k > kMaxK) return fail(HIPER_ERR_UNSUPPORTED, "k %d > %d", k, kMaxK);
  const bool pooled = ix->pooled;
  TRY(validate_queries(q_tokens, dtype, q_lens, n_q, q_max_len, dim, flags, pooled));
  if (n_q == 0) return HIPER_OK;
  if (out_keys ? !is_device_ptr(out_keys) : (!out_scores || !out_ids))
    return fail(HIPER_ERR_INVALID_ARG, "outputs are NULL");
  if (pooled)
    return pooled_search(ix, q_tokens, dtype, q_lens, n_q, dim, k, flags, comm, workspace,
                         workspace_bytes, out_scores, out_ids, nullptr, stream, out_keys);
  DevInfo di;
  TRY(device_info(di));
  if (di.device != ix->device) return fail(HIPER_ERR_INVALID_ARG, "index lives on device %d, current is %d", ix->device, di.device);
  KernelPlan kp;
  TRY(plan_kernel(di, n_q, q_max_len, index_slots(ix), index_slot_rows(ix), dim, kp, k));
  const int32_t world = comm ? comm->world : 1;
  TopkWs w;
  topk_ws_layout(n_q, dim, kp.n_q_pad, kp.n_parts, k, world, comm != nullptr, w);
  TRY(check_ws(workspace, workspace_bytes, w.total));
  uint8_t* ws = (uint8_t*)workspace;
  uint32_t* status = (uint32_t*)(ws + w.status);
  int32_t* qlens_dev = (int32_t*)(ws + w.qlens);
  __nv_bfloat16* qlayout = (__nv_bfloat16*)(ws + w.qlayout);
  uint64_t* partial = (uint64_t*)(ws + w.partial);
  uint32_t* progress = (uint32_t*)(ws + w.progress);

  // status = 0; lockstep words = ~0 ("not started": a pair that is not resident yet never holds the
  // others back, so the lockstep cannot deadlock even if the grid is not fully co-resident)
  CUDA_TRY(cudaMemsetAsync(status, 0, sizeof(uint32_t), stream));
  CUDA_TRY(cudaMemsetAsync(progress, 0xFF, w.qlens - w.progress, stream));
  TRY(prep_queries(q_tokens, dtype, q_lens, n_q, q_max_len, dim, flags, qlens_dev, qlayout, status, stream));
  if (flags & HIPER_VALIDATE_SYNC) TRY(sync_status(status, stream));

  if (kp.grid > 0) {
    alignas(64) CUtensorMap tq;
    TRY(make_tmap(&tq, qlayout, (int64_t)kp.n_q_pad * kp.qs, dim, 128));
    MaxsimArgs a = maxsim_args(kp, n_q, index_slots(ix), index_slot_rows(ix), dim, qlens_dev, ix->lens);
    a.k = k;
    set_packed_args(ix, a);
    a.id_base = ix->id_base;
    a.partial = partial;
    a.progress = getenv("HIPER_NO_LOCKSTEP") == nullptr ? progress : nullptr;
    // fewer row groups than pairs (small query batches) put ~pairs/G partitions in flight at once:
    // shrink the window so their lockstep footprint stays ~32 MB of L2 (measured at Q = 64:
    // window 64 vs 192 -> 578 vs 559 q/s)
    a.window = kLockstepWindow;
    const int slots = di.num_sms / 2;
    if (kp.n_groups < slots) {
      const int64_t slot_bytes = (int64_t)index_slot_rows(ix) * dim * 2;
      const int64_t w = ((int64_t)32 << 20) * kp.n_groups / ((int64_t)slots * slot_bytes);
      a.window = (int32_t)std::max<int64_t>(32, std::min<int64_t>(kLockstepWindow, w));
    }
    if (const char* e = getenv("HIPER_LOCKSTEP_WINDOW")) a.window = std::max(1, atoi(e));  // ablation
    TRY(launch_maxsim(1, k, kp, tq, ix->tmap_half, a, stream));
  }
  // partial lists [P][kEpiGroups][n_q_pad][k]: n_lists = P * kEpiGroups, each [n_q_pad][k]
  const int64_t q_stride = k, list_stride = (int64_t)kp.n_q_pad * k;
  const int32_t n_lists = kp.grid > 0 ? kp.n_parts * kEpiGroups : 0;
  if (out_keys)
    return launch_merge(partial, n_lists, list_stride, n_q, q_stride, k, out_keys, nullptr, nullptr, stream);
  if (!comm || comm->world == 1)
    return launch_merge(partial, n_lists, list_stride, n_q, q_stride, k, nullptr, out_scores, out_ids, stream);
  uint64_t* local = (uint64_t*)(ws + w.local);
  uint64_t* gathered = (uint64_t*)(ws + w.gathered);
  TRY(launch_merge(partial, n_lists, list_stride, n_q, q_stride, k, local, nullptr, nullptr, stream));
  return gather_merge(comm, local, gathered, n_q, k, out_scores, out_ids, stream);
}

extern "C" hiper_status hiper_maxsim_topk(const hiper_index* ix, const void* q_tokens,
                                          hiper_dtype dtype, const int32_t* q_lens, int32_t n_q,
                                          int32_t q_max_len, int32_t dim, int32_t k, uint32_t flags,
                                          const hiper_comm* comm, void* workspace,
                                          size_t workspace_bytes, float* out_scores,
                                          int64_t* out_ids, hiper_stream_t stream_) {
  g_launches = 0;
  HiperRange nv("hiper_maxsim_topk");
  return topk_search(ix, q_tokens, dtype, q_lens, n_q, q_max_len, dim, k, flags, comm, workspace,
                     workspace_bytes, out_scores, out_ids, nullptr, (cudaStream_t)stream_);
}

extern "C" hiper_status hiper_maxsim_topk_keys(const hiper_index* ix, const void* q_tokens,
                                               hiper_dtype dtype, const int32_t* q_lens, int32_t n_q,
                                               int32_t q_max_len, int32_t dim, int32_t k,
                                               uint32_t flags, void* workspace,
                                               size_t workspace_bytes, uint64_t* out_keys,
                                               hiper_stream_t stream_) {
  g_launches = 0;
  HiperRange nv("hiper_maxsim_topk_keys");
  if (!out_keys && n_q > 0) return fail(HIPER_ERR_INVALID_ARG, "out_keys is NULL");
  return topk_search(ix, q_tokens, dtype, q_lens, n_q, q_max_len, dim, k, flags, nullptr, workspace,
                     workspace_bytes, nullptr, nullptr, out_keys, (cudaStream_t)stream_);
}

// ============================================================================ dense scores
struct ScoresWs {
  size_t status = 0, qlens = 0, qlayout = 0, total = 0;
};
static void scores_ws_layout(int32_t n_q, int32_t dim, ScoresWs& w) {
  size_t off = 0;
  w.status = off;
  off += 256;
  w.qlens = off;
  off = align_up(off + (size_t)std::max(n_q, 1) * 4, 1024);
  w.qlayout = off;
  off = align_up(off + q_layout_bytes_max(n_q, dim), 1024);
  w.total = off;
}

extern "C" size_t hiper_maxsim_scores_workspace_size(const hiper_index* ix, int32_t n_q) {
  if (!ix || n_q < 0) return 0;
  if (ix->pooled) return pooled_ws_size(ix, n_q, 1, nullptr, false);
  ScoresWs w;
  scores_ws_layout(n_q, ix->dim, w);
  return w.total;
}

extern "C" hiper_status hiper_maxsim_scores(const hiper_index* ix, const void* q_tokens,
                                            hiper_dtype dtype, const int32_t* q_lens, int32_t n_q,
                                            int32_t q_max_len, int32_t dim, uint32_t flags,
                                            void* workspace, size_t workspace_bytes,
                                            float* out_scores, hiper_stream_t stream_) {
  g_launches = 0;
  HiperRange nv("hiper_maxsim_scores");
  cudaStream_t stream = (cudaStream_t)stream_;
  if (!ix) return fail(HIPER_ERR_INVALID_ARG, "index is NULL");
  if (dim != ix->dim) return fail(HIPER_ERR_DIM_MISMATCH, "query dim %d != index dim %d", dim, ix->dim);
  const bool pooled = ix->pooled;
  TRY(validate_queries(q_tokens, dtype, q_lens, n_q, q_max_len, dim, flags, pooled));
  if (n_q == 0 || ix->n == 0) return HIPER_OK;
  if (!out_scores) return fail(HIPER_ERR_INVALID_ARG, "out_scores is NULL");
  if (pooled)
    return pooled_search(ix, q_tokens, dtype, q_lens, n_q, dim, 1, flags, nullptr, workspace,
                         workspace_bytes, nullptr, nullptr, out_scores, stream);
  DevInfo di;
  TRY(device_info(di));
  KernelPlan kp;
  TRY(plan_kernel(di, n_q, q_max_len, index_slots(ix), index_slot_rows(ix), dim, kp));
  ScoresWs w;
  scores_ws_layout(n_q, dim, w);
  TRY(check_ws(workspace, workspace_bytes, w.total));
  uint8_t* ws = (uint8_t*)workspace;
  uint32_t* status = (uint32_t*)(ws + w.status);
  int32_t* qlens_dev = (int32_t*)(ws + w.qlens);
  __nv_bfloat16* qlayout = (__nv_bfloat16*)(ws + w.qlayout);
  CUDA_TRY(cudaMemsetAsync(status, 0, sizeof(uint32_t), stream));
  TRY(prep_queries(q_tokens, dtype, q_lens, n_q, q_max_len, dim, flags, qlens_dev, qlayout, status, stream));
  if (flags & HIPER_VALIDATE_SYNC) TRY(sync_status(status, stream));
  alignas(64) CUtensorMap tq;
  TRY(make_tmap(&tq, qlayout, (int64_t)kp.n_q_pad * kp.qs, dim, 128));
  MaxsimArgs a = maxsim_args(kp, n_q, index_slots(ix), index_slot_rows(ix), dim, qlens_dev, ix->lens);
  a.id_base = ix->id_base;
  a.scores = out_scores;
  a.score_ld = ix->n;
  set_packed_args(ix, a);
  return launch_maxsim(0, 1, kp, tq, ix->tmap_half, a, stream);
}

// ============================================================================ ColTrast scores + loss
struct ColtrastWs {
  size_t status = 0, qlens = 0, dlens = 0, pos = 0, rowloss = 0, qlayout = 0, dlayout = 0, scores = 0,
         total = 0;
};
static constexpr size_t kLossCounterOff = 4;  // u32 completion counter of the loss kernel (zeroed with status)
// The small host-fed region [status | qlens | dlens | pos] is contiguous so one staged copy fills it.
static void coltrast_ws_layout(int32_t n_q, int32_t n_d, int32_t d_max_len, int32_t dim, ColtrastWs& w) {
  const int32_t ld_pad = (int32_t)round_up(std::max(d_max_len, 1), 16);
  size_t off = 0;
  w.status = off;
  off += 16;
  w.qlens = off;
  off = align_up(off + (size_t)std::max(n_q, 1) * 4, 16);
  w.dlens = off;
  off = align_up(off + (size_t)std::max(n_d, 1) * 4, 16);
  w.pos = off;
  off = align_up(off + (size_t)std::max(n_q, 1) * 4, 256);
  w.rowloss = off;
  off = align_up(off + (size_t)std::max(n_q, 1) * 8, 1024);
  w.qlayout = off;
  off = align_up(off + q_layout_bytes_max(n_q, dim), 1024);
  w.dlayout = off;
  off = align_up(off + (size_t)std::max(n_d, 1) * ld_pad * dim * 2, 1024);
  w.scores = off;
  off = align_up(off + (size_t)std::max(n_q, 1) * std::max(n_d, 1) * 4, 1024);
  w.total = off;
}

// One staged H2D copy fills the small region of a ColTrast workspace: status = 0, query / doc
// lengths, positives (replaces a memset and up to three copies per step).
static hiper_status stage_small(const ColtrastWs& w, uint8_t* ws, const int32_t* q_lens, int32_t n_q,
                                const int32_t* d_lens, int32_t n_d, const int32_t* pos_idx,
                                cudaStream_t stream) {
  thread_local std::vector<uint8_t> host;
  host.assign(w.pos + (size_t)n_q * 4, 0);
  memcpy(host.data() + w.qlens, q_lens, (size_t)n_q * 4);
  memcpy(host.data() + w.dlens, d_lens, (size_t)n_d * 4);
  if (pos_idx) memcpy(host.data() + w.pos, pos_idx, (size_t)n_q * 4);
  return stage_h2d(ws + w.status, host.data(), pos_idx ? host.size() : w.pos, stream);
}

extern "C" size_t hiper_coltrast_workspace_size(int32_t n_q, int32_t n_d, int32_t d_max_len, int32_t dim) {
  if (n_q < 0 || n_d < 0 || dim <= 0) return 0;
  ColtrastWs w;
  coltrast_ws_layout(n_q, n_d, d_max_len, dim, w);
  return w.total;
}

// rows/counter (optional): the row-parallel kernel's scratch ([n_q] fp64, one zeroed u32 counter);
// without them one 1024-thread block does everything.
static hiper_status launch_loss(const float* S, int32_t n_q, int32_t n_d, int64_t ld,
                                const int32_t* pos_dev, float tau, float* out_loss,
                                cudaStream_t stream, const float* combine_with = nullptr,
                                float* out_combined = nullptr, double* rows = nullptr,
                                uint32_t* counter = nullptr, float* G = nullptr) {
  if (rows != nullptr && counter != nullptr && combine_with == nullptr) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)((n_q + 7) / 8));
    cfg.blockDim = dim3(256);
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;  // PDL (see launch_maxsim_t)
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    CUDA_TRY(cudaLaunchKernelEx(&cfg, infonce_rows_kernel, S, n_q, n_d, ld, pos_dev, tau, rows,
                                counter, out_loss, G));
  } else
    infonce_loss_kernel<<<1, 1024, 0, stream>>>(S, n_q, n_d, ld, pos_dev, tau, out_loss, combine_with,
                                                out_combined);
  CUDA_TRY(cudaGetLastError());
  ++g_launches;
  return HIPER_OK;
}

static hiper_status validate_loss_args(int32_t n_q, int32_t n_d, const int32_t* pos_idx, float tau) {
  if (n_q == 0) return fail(HIPER_ERR_EMPTY_BATCH, "empty batch");
  if (n_q < 0 || n_d < 0) return fail(HIPER_ERR_INVALID_ARG, "negative batch size");
  if (!(tau > 0.0f) || !std::isfinite(tau)) return fail(HIPER_ERR_BAD_TEMPERATURE, "temperature must be > 0 and finite");
  if (n_d == 0) return fail(HIPER_ERR_BAD_POSITIVE, "no candidates");
  if (pos_idx) {
    for (int32_t i = 0; i < n_q; ++i)
      if (pos_idx[i] < 0 || pos_idx[i] >= n_d)
        return fail(HIPER_ERR_BAD_POSITIVE, "pos_idx[%d] = %d outside 0..%d", i, pos_idx[i], n_d - 1);
  } else if (n_d < n_q) {
    return fail(HIPER_ERR_BAD_POSITIVE, "diagonal positives need n_d >= n_q");
  }
  return HIPER_OK;
}

extern "C" hiper_status hiper_coltrast_scores_loss(const void* q_tokens, const int32_t* q_lens, int32_t n_q,
                                                   int32_t q_max_len, const void* d_tokens,
                                                   const int32_t* d_lens, int32_t n_d, int32_t d_max_len,
                                                   int32_t dim, hiper_dtype dtype, uint32_t flags,
                                                   const int32_t* pos_idx, float temperature,
                                                   void* workspace, size_t workspace_bytes,
                                                   float* out_scores, float* out_loss, hiper_stream_t stream_) {
  g_launches = 0;
  HiperRange nv("hiper_coltrast_scores_loss");
  cudaStream_t stream = (cudaStream_t)stream_;
  TRY(validate_loss_args(n_q, n_d, pos_idx, temperature));
  TRY(validate_queries(q_tokens, dtype, q_lens, n_q, q_max_len, dim, flags));
  if (d_max_len < 1) return fail(HIPER_ERR_INVALID_ARG, "d_max_len must be >= 1");
  if (d_max_len > kMaxChunkLen) return fail(HIPER_ERR_UNSUPPORTED, "d_max_len %d > %d", d_max_len, kMaxChunkLen);
  TRY(check_lens(d_lens, n_d, d_max_len, "doc"));
  if (!d_tokens || !is_device_ptr(d_tokens) || ((uintptr_t)d_tokens & 15))
    return fail(HIPER_ERR_INVALID_ARG, "d_tokens must be 16-B aligned device memory");
  if (!out_loss) return fail(HIPER_ERR_INVALID_ARG, "out_loss is NULL");
  DevInfo di;
  TRY(device_info(di));
  const int32_t ld_pad = (int32_t)round_up(d_max_len, 16);
  KernelPlan kp;
  TRY(plan_kernel(di, n_q, q_max_len, n_d, ld_pad, dim, kp));
  ColtrastWs w;
  coltrast_ws_layout(n_q, n_d, d_max_len, dim, w);
  TRY(check_ws(workspace, workspace_bytes, w.total));
  uint8_t* ws = (uint8_t*)workspace;
  uint32_t* status = (uint32_t*)(ws + w.status);
  int32_t* qlens_dev = (int32_t*)(ws + w.qlens);
  int32_t* dlens_dev = (int32_t*)(ws + w.dlens);
  int32_t* pos_dev = (int32_t*)(ws + w.pos);
  __nv_bfloat16* qlayout = (__nv_bfloat16*)(ws + w.qlayout);
  __nv_bfloat16* dlayout = (__nv_bfloat16*)(ws + w.dlayout);
  float* S = out_scores ? out_scores : (float*)(ws + w.scores);

  TRY(stage_small(w, ws, q_lens, n_q, d_lens, n_d, pos_idx, stream));
  TRY(launch_norm2(q_tokens, n_q, q_max_len, qlens_dev, kp.n_q_pad, kp.qs, qlayout, d_tokens, n_d,
                   d_max_len, dlens_dev, n_d, ld_pad, dlayout, dtype, dim, flags, status, stream));
  if (flags & HIPER_VALIDATE_SYNC) TRY(sync_status(status, stream));

  alignas(64) CUtensorMap tq, td;
  TRY(make_tmap(&tq, qlayout, (int64_t)kp.n_q_pad * kp.qs, dim, 128));
  TRY(make_tmap(&td, dlayout, (int64_t)n_d * ld_pad, dim, (int32_t)kp.box_rows));
  MaxsimArgs a = maxsim_args(kp, n_q, n_d, ld_pad, dim, qlens_dev, dlens_dev);
  a.scores = S;
  a.score_ld = n_d;
  TRY(launch_maxsim(0, 1, kp, tq, td, a, stream));
  return launch_loss(S, n_q, n_d, n_d, pos_idx ? pos_dev : nullptr, temperature, out_loss, stream,
                     nullptr, nullptr, (double*)(ws + w.rowloss), (uint32_t*)(ws + w.status + kLossCounterOff));
}


// ============================================================================ N2: full ColTrast loss
// L = (L_LI + L_C) / 2:
//   L_LI  in-batch MaxSim InfoNCE over the local rank's b x b token-level scores (a10-a11);
//   L_C   InfoNCE (SimCSE form) over cos(pooled q_i, candidate_j) / tau_c, where the
//         candidates are the pooled passages of ALL ranks gathered with one ncclAllGather, local
//         positives first then the other ranks in (rank, position) order, truncated to
//         m = min(N, W) ("compared to min(N, W) samples").
// Pooled rows are NORM'd like token rows (cosine), scored by the pooled pair-GEMM kernel (MODE 0).
static hiper_status pooled_dense_raw(const DevInfo& di, const __nv_bfloat16* qlayout, int32_t n_q,
                                     const __nv_bfloat16* clayout, int64_t m, int32_t dim, float* S,
                                     int64_t ld, cudaStream_t stream) {
  PooledPlan pp;
  TRY(plan_pooled(di, n_q, m, pp, false));
  alignas(64) CUtensorMap tq, tc;
  TRY(make_tmap(&tq, qlayout, n_q, dim, 128));
  TRY(make_tmap(&tc, clayout, m, dim, 128));
  PooledArgs a{};
  a.n_q = n_q;
  a.n_qtiles = pp.n_qtiles;
  a.n_ctiles = pp.n_ctiles;
  a.n_parts = pp.n_parts;
  a.num_kb = num_kb_of(dim);
  a.k = 1;
  a.n_stages = pp.n_stages;
  a.stage_bytes = pp.stage_bytes;
  a.q_pad = pp.q_pad;
  a.n_chunks = m;
  a.scores = S;
  a.score_ld = ld;
  return launch_pooled<0>(pp, tq, tc, a, stream);
}

struct FullLossWs {
  size_t li = 0, ones = 0, qp = 0, dp = 0, gathered = 0, cand = 0, sc = 0, total = 0;
  size_t li_bytes = 0;
};
static void full_loss_ws_layout(int32_t b, int32_t d_max_len, int32_t dim, int32_t dp, int32_t m,
                                int32_t world, FullLossWs& w, int32_t n_ones = 0) {
  ColtrastWs cw;
  coltrast_ws_layout(b, b, d_max_len, dim, cw);
  size_t off = 0;
  w.li = off;
  w.li_bytes = cw.total;
  off = align_up(off + cw.total, 1024);
  w.ones = off;
  off = align_up(off + (size_t)std::max(std::max(b, n_ones), 1) * 4, 1024);
  w.qp = off;
  off = align_up(off + (size_t)std::max(b, 1) * dp * 2, 1024);
  w.dp = off;
  off = align_up(off + (size_t)std::max(b, 1) * dp * 2, 1024);
  w.gathered = off;
  off = align_up(off + (size_t)world * std::max(b, 1) * dp * 2, 1024);
  w.cand = off;
  off = align_up(off + (size_t)std::max(m, 1) * dp * 2, 1024);
  w.sc = off;
  off = align_up(off + (size_t)std::max(b, 1) * std::max(m, 1) * 4, 1024);
  w.total = off;
}

extern "C" size_t hiper_coltrast_loss_workspace_size(int32_t b, int32_t d_max_len, int32_t dim,
                                                     int32_t dp, int32_t n_max,
                                                     const hiper_comm* comm) {
  if (b < 0 || dim <= 0 || dp <= 0) return 0;
  const int32_t world = comm ? comm->world : 1;
  const int32_t m = (int32_t)std::min<int64_t>(std::max(n_max, 0), (int64_t)world * b);
  FullLossWs w;
  full_loss_ws_layout(b, d_max_len, dim, dp, m, world, w);
  return w.total;
}

static bool n2_force_nccl() {
  static const bool f = getenv("HIPER_N2_NCCL") != nullptr;  // A/B: the NCCL all-gather path
  return f;
}

// The full loss.  Exactly one of: comm (real ranks; the gather reads the peers' windows over NVLink,
// or NCCL when IPC is unavailable), sim_world > 0 (test support: d_pooled holds every simulated rank's
// passages [sim_world][b][dp] on this GPU and this call plays rank sim_rank), or neither (one rank).
static hiper_status coltrast_loss_impl(
    const void* q_tokens, const int32_t* q_lens, int32_t q_max_len, const void* d_tokens,
    const int32_t* d_lens, int32_t d_max_len, int32_t dim, const void* q_pooled,
    const void* d_pooled, int32_t dp, int32_t b, hiper_dtype dtype, uint32_t flags, int32_t n_max,
    float tau_li, float tau_c, hiper_comm_s* comm, int32_t sim_world, int32_t sim_rank,
    void* workspace, size_t workspace_bytes, float* out_losses, float* out_scores_c, int32_t* out_m,
    cudaStream_t stream) {
  if (b == 0) return fail(HIPER_ERR_EMPTY_BATCH, "empty batch");
  if (b < 0) return fail(HIPER_ERR_INVALID_ARG, "b < 0");
  if (n_max < b) return fail(HIPER_ERR_INVALID_ARG, "N (%d) < local batch (%d): positives must fit (SPEC NTooSmall)", n_max, b);
  if (!(tau_c > 0.0f) || !std::isfinite(tau_c) || !(tau_li > 0.0f) || !std::isfinite(tau_li))
    return fail(HIPER_ERR_BAD_TEMPERATURE, "temperatures must be > 0 and finite");
  TRY(check_dims(dp, true));
  if (!q_pooled || !d_pooled || !is_device_ptr(q_pooled) || !is_device_ptr(d_pooled) ||
      ((uintptr_t)q_pooled & 15) || ((uintptr_t)d_pooled & 15))
    return fail(HIPER_ERR_INVALID_ARG, "pooled inputs must be 16-B aligned device memory");
  if (!out_losses) return fail(HIPER_ERR_INVALID_ARG, "out_losses is NULL");
  const bool sim = sim_world > 0;
  if (sim && (sim_rank < 0 || sim_rank >= sim_world || sim_world > kMaxPeers))
    return fail(HIPER_ERR_INVALID_ARG, "simulated rank %d of %d (<= %d)", sim_rank, sim_world, kMaxPeers);
  const int32_t world = comm ? comm->world : (sim ? sim_world : 1);
  const int32_t rank = comm ? comm->rank : (sim ? sim_rank : 0);
  if (world > kMaxPeers) return fail(HIPER_ERR_UNSUPPORTED, "world %d > %d", world, kMaxPeers);
  const int32_t m = (int32_t)std::min<int64_t>(n_max, (int64_t)world * b);
  FullLossWs w;
  full_loss_ws_layout(b, d_max_len, dim, dp, m, world, w, sim ? world * b : b);
  TRY(check_ws(workspace, workspace_bytes, w.total));
  uint8_t* ws = (uint8_t*)workspace;
  DevInfo di;
  TRY(device_info(di));
  // L_LI on the local rank (writes out_losses[0])
  TRY(hiper_coltrast_scores_loss(q_tokens, q_lens, b, q_max_len, d_tokens, d_lens, b, d_max_len, dim,
                                 dtype, flags, nullptr, tau_li, ws + w.li, w.li_bytes, nullptr,
                                 out_losses, (hiper_stream_t)stream));
  int32_t launches = g_launches;
  // pooled rows -> NORM'd bf16 (the length array is all ones: one row per item)
  const int32_t n_norm = sim ? world * b : b;  // simulated: every rank's passages
  std::vector<int32_t> ones(n_norm, 1);
  int32_t* lens1 = (int32_t*)(ws + w.ones);
  __nv_bfloat16* qp = (__nv_bfloat16*)(ws + w.qp);
  __nv_bfloat16* dpp = (__nv_bfloat16*)(ws + w.dp);
  __nv_bfloat16* gathered = (__nv_bfloat16*)(ws + w.gathered);
  __nv_bfloat16* cand = (__nv_bfloat16*)(ws + w.cand);
  float* Sc = out_scores_c ? out_scores_c : (float*)(ws + w.sc);
  TRY(stage_h2d(lens1, ones.data(), (size_t)n_norm * 4, stream));
  uint32_t* status = (uint32_t*)(ws + w.li);  // the L_LI workspace's status word (same stream order)
  g_launches = 0;
  TRY(launch_norm(q_pooled, dtype, b, 1, lens1, b, 1, dp, flags, qp, status, stream));
  // candidates: local positives first, then the other ranks in (rank, position) order, m rows
  if (comm && world > 1 && !n2_force_nccl() && !comm->ipc_failed)
    TRY(peer_windows(comm, (size_t)b * dp * 2, stream));
  const bool windows = comm && world > 1 && !n2_force_nccl() && comm->win != nullptr;
  PeerGatherArgs ga{};
  ga.world = world;
  ga.rank = rank;
  ga.b = b;
  ga.dp = dp;
  ga.m = m;
  ga.cand = cand;
  if (windows) {
    // NORM straight into this rank's window of this epoch, publish it, read every peer's over NVLink
    const unsigned long long epoch = ++comm->epoch;
    const size_t par = kWinHeader + (size_t)(epoch & 1ull) * comm->win_bytes;
    TRY(launch_norm(d_pooled, dtype, b, 1, lens1, b, 1, dp, flags,
                    (__nv_bfloat16*)((uint8_t*)comm->win + par), status, stream));
    peer_signal_kernel<<<1, 1, 0, stream>>>((unsigned long long*)comm->win, epoch);
    CUDA_TRY(cudaGetLastError());
    ++g_launches;
    for (int32_t r = 0; r < world; ++r) {
      ga.src[r] = (const __nv_bfloat16*)((const uint8_t*)comm->peer[r] + par);
      ga.ready[r] = r == rank ? nullptr : (const unsigned long long*)comm->peer[r];
    }
    ga.epoch = epoch;
  } else if (sim) {
    TRY(launch_norm(d_pooled, dtype, n_norm, 1, lens1, n_norm, 1, dp, flags, gathered, status, stream));
    for (int32_t r = 0; r < world; ++r) ga.src[r] = gathered + (size_t)r * b * dp;
  } else if (world > 1) {  // NCCL: all-gather of every rank's NORM'd passages, then the same ordering
    TRY(launch_norm(d_pooled, dtype, b, 1, lens1, b, 1, dp, flags, dpp, status, stream));
    NCCL_TRY(ncclAllGather(dpp, gathered, (size_t)b * dp, ncclBfloat16, comm->comm, stream));
    TRY(nccl_async_check(comm, "ncclAllGather of pooled passages"));
    for (int32_t r = 0; r < world; ++r) ga.src[r] = gathered + (size_t)r * b * dp;
  } else {
    TRY(launch_norm(d_pooled, dtype, b, 1, lens1, b, 1, dp, flags, dpp, status, stream));
    ga.src[0] = dpp;
  }
  peer_gather_kernel<<<(unsigned)m, 128, 0, stream>>>(ga);
  CUDA_TRY(cudaGetLastError());
  ++g_launches;
  launches += g_launches;
  if (flags & HIPER_VALIDATE_SYNC) TRY(sync_status(status, stream));
  // L_C scores [b][m] and loss (writes out_losses[1] and out_losses[2] = (L_LI + L_C) / 2)
  g_launches = 0;
  TRY(pooled_dense_raw(di, qp, b, cand, m, dp, Sc, m, stream));
  TRY(launch_loss(Sc, b, m, m, nullptr, tau_c, out_losses + 1, stream, out_losses, out_losses + 2));
  g_launches += launches;
  if (out_m) *out_m = m;
  return HIPER_OK;
}

extern "C" hiper_status hiper_coltrast_loss(
    const void* q_tokens, const int32_t* q_lens, int32_t q_max_len, const void* d_tokens,
    const int32_t* d_lens, int32_t d_max_len, int32_t dim, const void* q_pooled,
    const void* d_pooled, int32_t dp, int32_t b, hiper_dtype dtype, uint32_t flags, int32_t n_max,
    float tau_li, float tau_c, const hiper_comm* comm, void* workspace, size_t workspace_bytes,
    float* out_losses, float* out_scores_c, int32_t* out_m, hiper_stream_t stream_) {
  g_launches = 0;
  HiperRange nv("hiper_coltrast_loss");
  return coltrast_loss_impl(q_tokens, q_lens, q_max_len, d_tokens, d_lens, d_max_len, dim, q_pooled,
                            d_pooled, dp, b, dtype, flags, n_max, tau_li, tau_c,
                            const_cast<hiper_comm_s*>(comm), 0, 0, workspace, workspace_bytes,
                            out_losses, out_scores_c, out_m, (cudaStream_t)stream_);
}

extern "C" size_t hiper_coltrast_loss_simulated_workspace_size(int32_t b, int32_t d_max_len,
                                                               int32_t dim, int32_t dp, int32_t n_max,
                                                               int32_t world) {
  if (b < 0 || dim <= 0 || dp <= 0 || world < 1) return 0;
  const int32_t m = (int32_t)std::min<int64_t>(std::max(n_max, 0), (int64_t)world * b);
  FullLossWs w;
  full_loss_ws_layout(b, d_max_len, dim, dp, m, world, w, world * b);
  return w.total;
}

extern "C" hiper_status hiper_coltrast_loss_simulated(
    const void* q_tokens, const int32_t* q_lens, int32_t q_max_len, const void* d_tokens,
    const int32_t* d_lens, int32_t d_max_len, int32_t dim, const void* q_pooled,
    const void* d_pooled_all, int32_t dp, int32_t b, hiper_dtype dtype, uint32_t flags,
    int32_t n_max, float tau_li, float tau_c, int32_t world, int32_t rank, void* workspace,
    size_t workspace_bytes, float* out_losses, float* out_scores_c, int32_t* out_m,
    hiper_stream_t stream_) {
  g_launches = 0;
  HiperRange nv("hiper_coltrast_loss_simulated");
  if (world < 1) return fail(HIPER_ERR_INVALID_ARG, "world < 1");
  return coltrast_loss_impl(q_tokens, q_lens, q_max_len, d_tokens, d_lens, d_max_len, dim, q_pooled,
                            d_pooled_all, dp, b, dtype, flags, n_max, tau_li, tau_c, nullptr, world,
                            rank, workspace, workspace_bytes, out_losses, out_scores_c, out_m,
                            (cudaStream_t)stream_);
}


// ============================================================================ N1: L_LI backward
struct GradWs {
  size_t base = 0, amax = 0, G = 0, ent = 0, bucket = 0, scratch = 0, qpart = 0, total = 0;
  int32_t S = 64, n_seg = 0;  // grad_d segments: hits per segment, segments per doc (at most)
  ColtrastWs cw;
};
static constexpr int32_t kGqRangesMax = 8;  // chunk ranges of the streamed grad_q (partials)
static void grad_ws_layout(int32_t n_q, int32_t n_d, int32_t d_max_len, int32_t dim, GradWs& w) {
  coltrast_ws_layout(n_q, n_d, d_max_len, dim, w.cw);
  const int32_t E = std::max(n_q, 1) * 32;
  w.S = 128;  // a power of two; segments per doc stay <= 128 (bounded scratch)
  if (const char* e = getenv("HIPER_GRAD_S")) w.S = std::max(64, std::min(1024, atoi(e)));
  while (w.S < E / 128) w.S *= 2;
  w.n_seg = (E + w.S - 1) / w.S;
  size_t off = align_up(w.cw.total, 1024);
  w.amax = off;
  off = align_up(off + (size_t)std::max(n_q, 1) * std::max(n_d, 1) * 32, 1024);
  w.G = off;
  off = align_up(off + (size_t)std::max(n_q, 1) * std::max(n_d, 1) * 4, 1024);
  w.ent = off;  // inverted argmax map per doc: [n_d][n_q * 32] {i * 32 + t, G_ij} + [n_d][258] starts
  off = align_up(off + (size_t)E * std::max(n_d, 1) * 8, 1024);
  w.bucket = off;
  off = align_up(off + (size_t)std::max(n_d, 1) * 258 * 4, 1024);
  w.scratch = off;  // [n_d][n_seg][2][dim] fp32 partials of rows that cross segments
  off = align_up(off + (size_t)std::max(n_d, 1) * w.n_seg * 2 * dim * 4, 1024);
  w.qpart = off;  // [R][n_q * 32][dim] fp32 partial sums of grad_q
  off = align_up(off + (size_t)kGqRangesMax * std::max(n_q, 1) * 32 * dim * 4, 1024);
  w.total = off;
}

extern "C" size_t hiper_coltrast_grad_workspace_size(int32_t n_q, int32_t n_d, int32_t d_max_len,
                                                     int32_t dim) {
  if (n_q < 0 || n_d < 0 || dim <= 0) return 0;
  GradWs w;
  grad_ws_layout(n_q, n_d, d_max_len, dim, w);
  return w.total;
}

// Programmatic dependent launch of a plain kernel: it may start while its stream predecessor
// drains and calls griddepcontrol.wait before touching that kernel's outputs (hides the launch gap
// between the short N1 backward kernels).
template <typename... KArgs, typename... Args>
static hiper_status launch_pdl(void (*kern)(KArgs...), unsigned grid, unsigned block, size_t smem,
                               cudaStream_t stream, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(block);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  static const bool off = getenv("HIPER_GRAD_PDL") && getenv("HIPER_GRAD_PDL")[0] == '0';  // A/B
  cfg.numAttrs = off ? 0 : 1;
  CUDA_TRY(cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...));
  return HIPER_OK;
}

// Fork/join onto a side stream (per host thread and device): grad_q and grad_d only share their
// inputs (G, the argmax map, the layouts), so they run concurrently.  Stream capture follows the
// fork/join (event record + wait), so the pattern is graph-capturable.  HIPER_GRAD_FORK=0: serial.
namespace {
struct SideStream {
  cudaStream_t s = nullptr;
  cudaEvent_t fork = nullptr, join = nullptr;
  ~SideStream() {  // at host-thread exit (errors ignored: the context may already be gone)
    if (fork) cudaEventDestroy(fork);
    if (join) cudaEventDestroy(join);
    if (s) cudaStreamDestroy(s);
    cudaGetLastError();
  }
};
}  // namespace
static hiper_status side_stream(int device, SideStream** out) {
  thread_local SideStream tab[16];
  if (device < 0 || device >= 16) return fail(HIPER_ERR_UNSUPPORTED, "device %d", device);
  SideStream& ss = tab[device];
  if (!ss.s) {
    CUDA_TRY(cudaStreamCreateWithFlags(&ss.s, cudaStreamNonBlocking));
    CUDA_TRY(cudaEventCreateWithFlags(&ss.fork, cudaEventDisableTiming));
    CUDA_TRY(cudaEventCreateWithFlags(&ss.join, cudaEventDisableTiming));
  }
  *out = &ss;
  return HIPER_OK;
}

extern "C" hiper_status hiper_coltrast_scores_loss_grad(
    const void* q_tokens, const int32_t* q_lens, int32_t n_q, int32_t q_max_len, const void* d_tokens,
    const int32_t* d_lens, int32_t n_d, int32_t d_max_len, int32_t dim, hiper_dtype dtype,
    uint32_t flags, const int32_t* pos_idx, float temperature, void* workspace,
    size_t workspace_bytes, float* out_scores, float* out_loss, float* grad_q, float* grad_d,
    hiper_stream_t stream_) {
  g_launches = 0;
  HiperRange nv("hiper_coltrast_scores_loss_grad");
  cudaStream_t stream = (cudaStream_t)stream_;
  TRY(validate_loss_args(n_q, n_d, pos_idx, temperature));
  TRY(validate_queries(q_tokens, dtype, q_lens, n_q, q_max_len, dim, flags));
  if (d_max_len < 1) return fail(HIPER_ERR_INVALID_ARG, "d_max_len must be >= 1");
  if (d_max_len > 256 || q_max_len > 32 || (dim != 64 && dim != 128))
    return fail(HIPER_ERR_UNSUPPORTED, "backward supports q_max_len <= 32, d_max_len <= 256, dim 64 or 128");
  TRY(check_lens(d_lens, n_d, d_max_len, "doc"));
  if (!d_tokens || !is_device_ptr(d_tokens) || ((uintptr_t)d_tokens & 15))
    return fail(HIPER_ERR_INVALID_ARG, "d_tokens must be 16-B aligned device memory");
  if (!out_loss || !grad_q || !grad_d) return fail(HIPER_ERR_INVALID_ARG, "outputs are NULL");
  DevInfo di;
  TRY(device_info(di));
  const int32_t ld_pad = (int32_t)round_up(d_max_len, 16);
  KernelPlan kp;
  TRY(plan_kernel(di, n_q, q_max_len, n_d, ld_pad, dim, kp));
  if (n_q > 2048) return fail(HIPER_ERR_UNSUPPORTED, "backward supports n_q <= 2048 (got %d)", n_q);
  GradWs w;
  grad_ws_layout(n_q, n_d, d_max_len, dim, w);
  TRY(check_ws(workspace, workspace_bytes, w.total));
  uint8_t* ws = (uint8_t*)workspace;
  const ColtrastWs& c = w.cw;
  uint32_t* status = (uint32_t*)(ws + c.status);
  int32_t* qlens_dev = (int32_t*)(ws + c.qlens);
  int32_t* dlens_dev = (int32_t*)(ws + c.dlens);
  int32_t* pos_dev = (int32_t*)(ws + c.pos);
  __nv_bfloat16* qlayout = (__nv_bfloat16*)(ws + c.qlayout);
  __nv_bfloat16* dlayout = (__nv_bfloat16*)(ws + c.dlayout);
  float* S = out_scores ? out_scores : (float*)(ws + c.scores);
  uint8_t* amax = ws + w.amax;
  float* G = (float*)(ws + w.G);

  TRY(stage_small(c, ws, q_lens, n_q, d_lens, n_d, pos_idx, stream));
  TRY(launch_norm2(q_tokens, n_q, q_max_len, qlens_dev, kp.n_q_pad, kp.qs, qlayout, d_tokens, n_d,
                   d_max_len, dlens_dev, n_d, ld_pad, dlayout, dtype, dim, flags, status, stream));
  if (flags & HIPER_VALIDATE_SYNC) TRY(sync_status(status, stream));
  alignas(64) CUtensorMap tq, td;
  TRY(make_tmap(&tq, qlayout, (int64_t)kp.n_q_pad * kp.qs, dim, 128));
  TRY(make_tmap(&td, dlayout, (int64_t)n_d * ld_pad, dim, (int32_t)kp.box_rows));
  MaxsimArgs a = maxsim_args(kp, n_q, n_d, ld_pad, dim, qlens_dev, dlens_dev);
  a.scores = S;
  a.score_ld = n_d;
  a.amax = amax;
  TRY(launch_maxsim(2, 1, kp, tq, td, a, stream));                       // S + argmax (a3-a5)
  const int32_t* pd = pos_idx ? pos_dev : nullptr;
  // a11 and G = dL_LI/dS in one launch (the row warps write their row of G)
  TRY(launch_loss(S, n_q, n_d, n_d, pd, temperature, out_loss, stream, nullptr, nullptr,
                  (double*)(ws + c.rowloss), (uint32_t*)(ws + c.status + kLossCounterOff), G));
  const uint32_t an = (flags & HIPER_ASSUME_NORMALIZED) ? 1u : 0u;
  const int64_t qrows = (int64_t)n_q * q_max_len;
  const unsigned qblocks = (unsigned)((qrows + 7) / 8);
  const size_t dsmem = (size_t)n_q * 32 * 3 + (size_t)n_q * 8 + 2 * kSortWarps * 257 * 4;
  // grad_q: chunk tiles streamed through shared memory per 8 queries (partials over R chunk ranges)
  const int32_t qblk = (n_q + kGqWarps - 1) / kGqWarps;
  const int32_t R = std::max(1, std::min({kGqRangesMax, n_d, di.num_sms / std::max(qblk, 1)}));
  alignas(64) CUtensorMap tdg;  // doc rows as 64-dim x ld_pad boxes
  TRY(make_tmap(&tdg, dlayout, (int64_t)n_d * ld_pad, dim, ld_pad));
  float* qpart = (float*)(ws + w.qpart);
  auto launch_grads = [&](auto vpl, auto tin) -> hiper_status {
    constexpr int VPL = decltype(vpl)::value;
    using Tin = decltype(tin);
    auto gqs = grad_q_stream_kernel<VPL / 2>;
    const int gstage = ld_pad * 128 * (VPL / 2);
    const int gns = std::max(2, std::min(4, (di.max_smem - 1024 - 128) / gstage));  // TMA ring depth
    const int gsm = 1024 + gns * gstage + 128;
    CUDA_TRY(set_max_smem((const void*)gqs, gsm));
    const char* ef = getenv("HIPER_GRAD_FORK");
    SideStream* ss = nullptr;
    if (!(ef && ef[0] == '0')) TRY(side_stream(di.device, &ss));
    cudaStream_t qs = stream;
    if (ss) {  // grad_q on the side stream, grad_d on the caller's
      CUDA_TRY(cudaEventRecord(ss->fork, stream));
      CUDA_TRY(cudaStreamWaitEvent(ss->s, ss->fork, 0));
      qs = ss->s;
    }
    gqs<<<(unsigned)(qblk * R), (kGqWarps + 1) * 32, gsm, qs>>>(tdg, G, amax, n_q, n_d, ld_pad,
                                                                qlens_dev, R, qpart, gns);
    CUDA_TRY(cudaGetLastError());
    TRY(launch_pdl(grad_q_reduce_kernel<VPL, Tin>, qblocks, 256, 0, qs, (const float*)qpart, R, n_q,
                   (const Tin*)q_tokens, q_max_len, (const int32_t*)qlens_dev, an, grad_q));
    if (ss) CUDA_TRY(cudaEventRecord(ss->join, ss->s));
    g_launches += 1;
    // grad_d: the inverted argmax map per doc (one block per doc), then one warp per segment of S
    // sorted hits, so "hub" doc rows that take most argmax hits are spread over many warps.
    CUDA_TRY(set_max_smem((const void*)grad_d_sort_kernel, (int)dsmem));
    uint2* ent = (uint2*)(ws + w.ent);
    int32_t* bkt = (int32_t*)(ws + w.bucket);
    TRY(launch_pdl(grad_d_sort_kernel, (unsigned)n_d, kSortWarps * 32, dsmem, stream,
                   (const uint8_t*)amax, (const float*)G, n_q, n_d, (const int32_t*)qlens_dev, ent, bkt));
    const int64_t sblocks = (int64_t)n_d * ((w.n_seg + 7) / 8);
    float* scr = (float*)(ws + w.scratch);
    TRY(launch_pdl(grad_d_seg_kernel<VPL>, (unsigned)sblocks, 256, 0, stream, n_q,
                   (const __nv_bfloat16*)qlayout, (const uint2*)ent, (const int32_t*)bkt,
                   (int32_t)__builtin_ctz((unsigned)w.S), (int32_t)w.n_seg, scr, d_max_len, grad_d));
    const int64_t fwarps = (int64_t)n_d * ((d_max_len + 3) / 4);  // 4 rows per warp
    TRY(launch_pdl(grad_d_finish_kernel<VPL, Tin>, (unsigned)((fwarps + 7) / 8), 256, 0, stream,
                   (const int32_t*)bkt, (int32_t)__builtin_ctz((unsigned)w.S), (int32_t)w.n_seg,
                   (const float*)scr, n_d, (const Tin*)d_tokens, d_max_len, (const int32_t*)dlens_dev,
                   an, grad_d));
    if (ss) CUDA_TRY(cudaStreamWaitEvent(stream, ss->join, 0));  // join: the call ends on `stream`
    g_launches += 4;
    return HIPER_OK;
  };
  using I2 = std::integral_constant<int, 2>;
  using I4 = std::integral_constant<int, 4>;
  if (dim == 128) {
    if (dtype == HIPER_F32) return launch_grads(I4{}, float{});
    return launch_grads(I4{}, __nv_bfloat16{});
  }
  if (dtype == HIPER_F32) return launch_grads(I2{}, float{});
  return launch_grads(I2{}, __nv_bfloat16{});
}


// ============================================================================ N3: two-stage retrieval
// Stage 1: pooled cosine top-K1 (the paper's deployed retrieval) on a pooled
// index; stage 2: exact MaxSim re-scoring of each query's own K1 candidates on the token index of the
// same chunks (ColBERTv2's pattern; SPEC.md:268-276 rerank), final top-k.  Stage 2 is
// the gather kernel of kernels/rerank_gather.cuh: Q * K1 (query, candidate) pairs, each computed
// once, HBM-bound on the candidates' rows.
struct TwoStageWs {
  size_t pooled = 0, pooled_bytes = 0, s1_scores = 0, s1_ids = 0, slots = 0, status = 0, qlens = 0,
         qlayout = 0, S2 = 0, local = 0, gathered = 0, total = 0;
};
static constexpr int32_t kRerankMaxDim = 128, kRerankMaxQueryLen = 32;
static void two_stage_ws_layout(const hiper_index* pix, const hiper_index* tix, int32_t n_q,
                                int32_t k1, int32_t k, const hiper_comm* comm, TwoStageWs& w) {
  size_t off = 0;
  w.pooled = off;
  w.pooled_bytes = pooled_ws_size(pix, n_q, k1, comm, true);
  off = align_up(off + w.pooled_bytes, 1024);
  w.s1_scores = off;
  off = align_up(off + (size_t)std::max(n_q, 1) * k1 * 4, 256);
  w.s1_ids = off;
  off = align_up(off + (size_t)std::max(n_q, 1) * k1 * 8, 256);
  w.slots = off;
  off = align_up(off + (size_t)std::max(n_q, 1) * k1 * 4, 256);
  w.status = off;
  off += 256;
  w.qlens = off;
  off = align_up(off + (size_t)std::max(n_q, 1) * 4, 1024);
  w.qlayout = off;
  off = align_up(off + (size_t)n_q_pad_of(n_q) * 32 * tix->dim * 2, 1024);
  w.S2 = off;
  off = align_up(off + (size_t)std::max(n_q, 1) * k1 * 4, 1024);
  w.local = off;  // multi-rank: this rank's re-scored top-k keys, then every rank's
  if (comm) off = align_up(off + (size_t)std::max(n_q, 1) * k * 8, 256);
  w.gathered = off;
  if (comm) off = align_up(off + (size_t)comm->world * std::max(n_q, 1) * k * 8, 256);
  w.total = off;
}

extern "C" size_t hiper_two_stage_workspace_size(const hiper_index* pooled_idx,
                                                 const hiper_index* token_idx, int32_t n_q,
                                                 int32_t k1, const hiper_comm* comm) {
  if (!pooled_idx || !token_idx || n_q < 0 || k1 < 1) return 0;
  TwoStageWs w;
  two_stage_ws_layout(pooled_idx, token_idx, n_q, k1, k1, comm, w);  // k <= k1
  return w.total;
}

template <int KR>
static hiper_status launch_rerank_select(const float* S2, const int32_t* slots, int32_t k1, int32_t n_q,
                                         int64_t id_base, int32_t k, float* out_scores,
                                         int64_t* out_ids, uint64_t* out_keys, cudaStream_t stream) {
  rerank_select_kernel<KR><<<(n_q + 7) / 8, 256, 0, stream>>>(S2, slots, k1, n_q, id_base, k, out_scores,
                                                             out_ids, out_keys);
  CUDA_TRY(cudaGetLastError());
  ++g_launches;
  return HIPER_OK;
}

extern "C" hiper_status hiper_two_stage_topk(const hiper_index* pix, const hiper_index* tix,
                                             const void* q_pooled, const void* q_tokens,
                                             hiper_dtype dtype, const int32_t* q_lens, int32_t n_q,
                                             int32_t q_max_len, int32_t k1, int32_t k,
                                             uint32_t flags, const hiper_comm* comm, void* workspace,
                                             size_t workspace_bytes, float* out_scores,
                                             int64_t* out_ids, hiper_stream_t stream_) {
  g_launches = 0;
  HiperRange nv("hiper_two_stage_topk");
  cudaStream_t stream = (cudaStream_t)stream_;
  if (!pix || !tix) return fail(HIPER_ERR_INVALID_ARG, "index is NULL");
  if (!pix->pooled) return fail(HIPER_ERR_INVALID_ARG, "stage-1 index must be pooled (HIPER_POOLED)");
  if (tix->pooled) return fail(HIPER_ERR_INVALID_ARG, "stage-2 index must hold token rows");
  if (pix->n != tix->n || pix->id_base != tix->id_base)
    return fail(HIPER_ERR_INVALID_ARG, "the two indexes must cover the same chunks (n, id_base)");
  if (k1 < 1 || k < 1 || k > k1) return fail(HIPER_ERR_INVALID_ARG, "need 1 <= k <= k1");
  if (k1 > kMaxK) return fail(HIPER_ERR_UNSUPPORTED, "k1 %d > %d", k1, kMaxK);
  if (tix->dim > kRerankMaxDim || q_max_len > kRerankMaxQueryLen || tix->max_len > 256)
    return fail(HIPER_ERR_UNSUPPORTED, "rerank supports token dim <= %d, q_max_len <= %d, max_len <= 256",
                kRerankMaxDim, kRerankMaxQueryLen);
  {
    std::vector<int32_t> ones(std::max(n_q, 0), 1);
    TRY(validate_queries(q_pooled, dtype, ones.data(), n_q, 1, pix->dim, flags, true));
  }
  TRY(validate_queries(q_tokens, dtype, q_lens, n_q, q_max_len, tix->dim, flags));
  if (n_q == 0) return HIPER_OK;
  if (!out_scores || !out_ids) return fail(HIPER_ERR_INVALID_ARG, "outputs are NULL");
  DevInfo di;
  TRY(device_info(di));
  TwoStageWs w;
  two_stage_ws_layout(pix, tix, n_q, k1, k, comm, w);
  TRY(check_ws(workspace, workspace_bytes, w.total));
  const bool multi = comm != nullptr && comm->world > 1;
  uint8_t* ws = (uint8_t*)workspace;
  float* s1s = (float*)(ws + w.s1_scores);
  int64_t* s1i = (int64_t*)(ws + w.s1_ids);
  int32_t* slots = (int32_t*)(ws + w.slots);
  // stage 1: pooled top-k1 (pooled queries have one row each; lengths all 1)
  // (with comm: the GLOBAL pooled top-k1, identical on every rank)
  std::vector<int32_t> ones(n_q, 1);
  TRY(pooled_search(pix, q_pooled, dtype, ones.data(), n_q, pix->dim, k1, flags, comm,
                    ws + w.pooled, w.pooled_bytes, s1s, s1i, nullptr, stream));
  int32_t launches = g_launches;
  g_launches = 0;
  // stage 2: this shard's slots, token query prep, the gather-MaxSim of every (query, own candidate)
  const int64_t n_items = (int64_t)n_q * k1;
  ids_to_slots_kernel<<<(unsigned)((n_items + 255) / 256), 256, 0, stream>>>(s1i, n_items, pix->id_base,
                                                                            pix->n, slots);
  CUDA_TRY(cudaGetLastError());
  ++g_launches;
  uint32_t* status = (uint32_t*)(ws + w.status);
  int32_t* qlens_dev = (int32_t*)(ws + w.qlens);
  __nv_bfloat16* qlayout = (__nv_bfloat16*)(ws + w.qlayout);
  float* S2 = (float*)(ws + w.S2);
  CUDA_TRY(cudaMemsetAsync(status, 0, sizeof(uint32_t), stream));
  TRY(prep_queries(q_tokens, dtype, q_lens, n_q, q_max_len, tix->dim, flags, qlens_dev, qlayout,
                   status, stream));
  if (flags & HIPER_VALIDATE_SYNC) TRY(sync_status(status, stream));
  // an empty shard has no token rows and no candidates (every slot is -1): skip the gather, but
  // still take part in the all-gather below
  if (tix->n > 0) {
    // the token index as 64-dim x 64-row and x 16-row boxes (only roundup(len, 16) rows fetched)
    alignas(64) CUtensorMap t64, t16;
    const int64_t trows = tix->packed ? tix->n_rows : tix->n * (int64_t)tix->ld_pad;
    TRY(make_tmap(&t64, tix->tok, trows, tix->dim, 64));
    TRY(make_tmap(&t16, tix->tok, trows, tix->dim, 16));
    RerankArgs ra{};
    ra.qlay = qlayout;
    ra.q_lens = qlens_dev;
    ra.slots = slots;
    ra.d_lens = tix->lens;
    ra.row_of = tix->packed ? tix->row_of : nullptr;
    ra.ld_pad = tix->ld_pad;
    ra.dim = tix->dim;
    ra.k1 = k1;
    ra.n_items = n_items;
    ra.n_index = tix->n;
    ra.S2 = S2;
    auto kern = num_kb_of(tix->dim) == 1 ? rerank_gather_kernel<1, 6> : rerank_gather_kernel<2, 3>;
    const int smem = 1024 + kRerankWarps * (num_kb_of(tix->dim) == 1 ? 6 : 3) * 64 * 128 * num_kb_of(tix->dim) + 256;
    CUDA_TRY(set_max_smem((const void*)kern, smem));
    const int64_t want = (n_items + 3) / 4;  // at least ~4 items per warp
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(di.num_sms, want / kRerankWarps));
    ProfTicket ev;
    TRY(profile_begin(stream, HIPER_PROF_RERANK, &ev));
    kern<<<grid, kRerankWarps * 32, smem, stream>>>(t64, t16, ra);
    CUDA_TRY(cudaGetLastError());
    TRY(profile_end(stream, ev));
    ++g_launches;
  }
  uint64_t* local = multi ? (uint64_t*)(ws + w.local) : nullptr;
  float* os = multi ? nullptr : out_scores;
  int64_t* oi = multi ? nullptr : out_ids;
  if (k <= 32) TRY(launch_rerank_select<1>(S2, slots, k1, n_q, tix->id_base, k, os, oi, local, stream));
  else if (k <= 64) TRY(launch_rerank_select<2>(S2, slots, k1, n_q, tix->id_base, k, os, oi, local, stream));
  else TRY(launch_rerank_select<4>(S2, slots, k1, n_q, tix->id_base, k, os, oi, local, stream));
  // multi-rank: every rank re-scored the candidates it owns; one all-gather of the re-scored top-k
  // keys and the same merge on every rank (keys are unique: bitwise the 1-GPU answer)
  if (multi) TRY(gather_merge(comm, local, (uint64_t*)(ws + w.gathered), n_q, k, out_scores, out_ids, stream));
  g_launches += launches;
  return HIPER_OK;
}

extern "C" hiper_status hiper_infonce_loss(const float* scores, int32_t n_q, int32_t n_d,
                                           const int32_t* pos_idx, float temperature, void* workspace,
                                           size_t workspace_bytes, float* out_loss, hiper_stream_t stream_) {
  g_launches = 0;
  HiperRange nv("hiper_infonce_loss");
  cudaStream_t stream = (cudaStream_t)stream_;
  TRY(validate_loss_args(n_q, n_d, pos_idx, temperature));
  if (!scores || !out_loss) return fail(HIPER_ERR_INVALID_ARG, "NULL pointer");
  const size_t need = align_up((size_t)n_q * 4, 1024);
  if (pos_idx) TRY(check_ws(workspace, workspace_bytes, need));
  if (pos_idx) TRY(stage_h2d(workspace, pos_idx, (size_t)n_q * 4, stream));
  return launch_loss(scores, n_q, n_d, n_d, pos_idx ? (const int32_t*)workspace : nullptr, temperature,
                     out_loss, stream);
}
