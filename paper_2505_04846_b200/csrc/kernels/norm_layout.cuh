// norm_layout.cuh -- steps a1 (corpus layout) and a2 (query preparation).
//
// One thread per OUTPUT row.  Row j < len of item i: NORM (R1, "rows normalized on entry",
// SPEC.md:285):
//   acc = 0; for k ascending: acc = fma_rn(x_k, x_k, acc);  inv = 1 / sqrt(acc) (both RN);
//   y_k = RNE_bf16(x_k * inv)
// Rows j >= len (and items >= n_items) are written as zero rows.  The layout step is HBM-bound
// (read d*in_bytes, write d*2 bytes per row); the per-thread sequential fma chain keeps the
// summation order fixed so the result is bit-identical to the oracle's independent NORM.
#pragma once
#include <cuda_bf16.h>
#include <cstdint>

namespace hiper {

constexpr uint32_t kStatusZeroRow = 1u;
constexpr uint32_t kStatusNonFinite = 2u;

__device__ __forceinline__ float load_elem(const float* p) { return *p; }
__device__ __forceinline__ float load_elem(const __nv_bfloat16* p) { return __bfloat162float(*p); }

template <typename Tin>
__device__ __forceinline__ void load8(const Tin* p, float (&x)[8]);
template <>
__device__ __forceinline__ void load8<float>(const float* p, float (&x)[8]) {
  const float4 a = *reinterpret_cast<const float4*>(p);
  const float4 b = *reinterpret_cast<const float4*>(p + 4);
  x[0] = a.x; x[1] = a.y; x[2] = a.z; x[3] = a.w;
  x[4] = b.x; x[5] = b.y; x[6] = b.z; x[7] = b.w;
}
template <>
__device__ __forceinline__ void load8<__nv_bfloat16>(const __nv_bfloat16* p, float (&x)[8]) {
  const uint4 u = *reinterpret_cast<const uint4*>(p);
  const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    x[2 * i] = __uint_as_float(w[i] << 16);
    x[2 * i + 1] = __uint_as_float(w[i] & 0xFFFF0000u);
  }
}

// in:  [n_src][in_rows][d] (element strides), only items < n_src / rows < lens[item] are read
// out: [n_items][out_rows][d] bf16
// lens: device [n_src] (items >= n_src are empty)
// d % 8 == 0 and 16-B aligned rows.  In-place (in == out) is allowed when Tin == bf16 and
// in_rows == out_rows: every thread reads and writes only its own row.
// dst_row (packed layout, N4; nullptr = dense): item i's rows go to packed rows dst_row[i] + j for
// j < roundup(len, 16) only (the padding rows of its 16-row slot are zeroed here, then replaced by
// copies of its last real row by pack_pad_replicate_kernel); out_rows is then just
// the per-item thread range (>= roundup(max_len, 16)).
template <typename Tin>
__device__ __forceinline__ void norm_row(int64_t row, const Tin* in, int64_t n_src, int32_t in_rows,
                                         const int32_t* __restrict__ lens, int64_t n_items,
                                         int32_t out_rows, int32_t d, uint32_t assume_normalized,
                                         uint32_t check_finite, __nv_bfloat16* out, uint32_t* status,
                                         const int64_t* __restrict__ dst_row) {
  if (row >= n_items * (int64_t)out_rows) return;
  const int64_t item = row / out_rows;
  const int32_t j = (int32_t)(row - item * out_rows);
  const int32_t len = item < n_src ? lens[item] : 0;
  if (dst_row != nullptr && j >= ((len + 15) & ~15)) return;
  uint4* dst = reinterpret_cast<uint4*>(out + (dst_row != nullptr ? dst_row[item] + j : row) * d);
  if (j >= len) {
    for (int32_t k = 0; k < d; k += 8) dst[k / 8] = make_uint4(0, 0, 0, 0);
    return;
  }
  const Tin* src = in + (item * in_rows + j) * (int64_t)d;
  float inv = 1.0f;
  if (!assume_normalized) {
    float acc = 0.0f;
    bool finite = true;
    for (int32_t k = 0; k < d; k += 8) {
      float x[8];
      load8<Tin>(src + k, x);
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        finite &= isfinite(x[i]);
        acc = __fmaf_rn(x[i], x[i], acc);
      }
    }
    if (!finite) {
      if (status) atomicOr(status, kStatusNonFinite);
    } else if (acc == 0.0f) {
      if (status) atomicOr(status, kStatusZeroRow);
    }
    inv = __fdiv_rn(1.0f, __fsqrt_rn(acc));
  } else if (check_finite) {
    bool finite = true;
    for (int32_t k = 0; k < d; k += 8) {
      float x[8];
      load8<Tin>(src + k, x);
#pragma unroll
      for (int i = 0; i < 8; ++i) finite &= isfinite(x[i]);
    }
    if (!finite && status) atomicOr(status, kStatusNonFinite);
  }
  for (int32_t k = 0; k < d; k += 8) {
    float x[8];
    load8<Tin>(src + k, x);
    uint32_t w[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const float a = assume_normalized ? x[2 * i] : __fmul_rn(x[2 * i], inv);
      const float b = assume_normalized ? x[2 * i + 1] : __fmul_rn(x[2 * i + 1], inv);
      const __nv_bfloat16 ha = __float2bfloat16_rn(a);
      const __nv_bfloat16 hb = __float2bfloat16_rn(b);
      w[i] = (uint32_t)__bfloat16_as_ushort(ha) | ((uint32_t)__bfloat16_as_ushort(hb) << 16);
    }
    dst[k / 8] = make_uint4(w[0], w[1], w[2], w[3]);
  }
}

template <typename Tin>
__global__ void __launch_bounds__(256) norm_layout_kernel(const Tin* in, int64_t n_src, int32_t in_rows,
                                                          const int32_t* __restrict__ lens,
                                                          int64_t n_items, int32_t out_rows, int32_t d,
                                                          uint32_t assume_normalized,
                                                          uint32_t check_finite,
                                                          __nv_bfloat16* out, uint32_t* status,
                                                          const int64_t* __restrict__ dst_row) {
  norm_row<Tin>((int64_t)blockIdx.x * blockDim.x + threadIdx.x, in, n_src, in_rows, lens, n_items,
                out_rows, d, assume_normalized, check_finite, out, status, dst_row);
}

// Same NORM with TPR = d/16 threads per row (d <= 512): each lane owns 16 consecutive elements, the
// loads and stores are coalesced, and the fp32 fma chain still runs over k in ascending order -- lane t
// continues the accumulator it receives from lane t-1 -- so the result is bit-identical to the
// one-thread-per-row form above.
template <typename Tin>
__device__ __forceinline__ void load16(const Tin* p, float (&x)[16]) {
  float a[8], b[8];
  load8<Tin>(p, a);
  load8<Tin>(p + 8, b);
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    x[i] = a[i];
    x[8 + i] = b[i];
  }
}
template <typename Tin, int TPR>
__device__ __forceinline__ void norm_row_group(int64_t row, uint32_t sub, const Tin* in, int64_t n_src,
                                               int32_t in_rows, const int32_t* __restrict__ lens,
                                               int64_t n_items, int32_t out_rows, int32_t d,
                                               uint32_t assume_normalized, uint32_t check_finite,
                                               __nv_bfloat16* out, uint32_t* status,
                                               const int64_t* __restrict__ dst_row) {
  const bool in_range = row < n_items * (int64_t)out_rows;
  int64_t item = 0;
  int32_t j = 0, len = 0;
  bool write = false, real = false;
  if (in_range) {
    item = row / out_rows;
    j = (int32_t)(row - item * out_rows);
    len = item < n_src ? lens[item] : 0;
    write = !(dst_row != nullptr && j >= ((len + 15) & ~15));
    real = j < len;
  }
  float x[16];
  if (real) {
    // in == out with dst_row set: a caller-packed buffer normalised in place (HIPER_PACKED |
    // HIPER_BORROW_TOKENS); each lane reads, then writes, only its own 16 elements
    const int64_t src_row = (dst_row != nullptr && (const void*)in == (const void*)out)
                                ? dst_row[item] + j
                                : item * in_rows + j;
    load16<Tin>(in + src_row * (int64_t)d + sub * 16, x);
  } else {
#pragma unroll
    for (int i = 0; i < 16; ++i) x[i] = 0.0f;
  }
  bool finite = true;
#pragma unroll
  for (int i = 0; i < 16; ++i) finite &= isfinite(x[i]);
  uint32_t nonfinite = finite ? 0u : 1u;
#pragma unroll
  for (int o = TPR / 2; o >= 1; o >>= 1) nonfinite |= __shfl_xor_sync(0xffffffffu, nonfinite, o, TPR);
  float acc = 0.0f;
  if (!assume_normalized) {
#pragma unroll
    for (int t = 0; t < TPR; ++t) {
      if (sub == (uint32_t)t) {
#pragma unroll
        for (int i = 0; i < 16; ++i) acc = __fmaf_rn(x[i], x[i], acc);
      }
      acc = __shfl_sync(0xffffffffu, acc, t, TPR);
    }
  }
  if (real && sub == 0 && status != nullptr) {
    if (!assume_normalized) {
      if (nonfinite) atomicOr(status, kStatusNonFinite);
      else if (acc == 0.0f) atomicOr(status, kStatusZeroRow);
    } else if (check_finite && nonfinite) {
      atomicOr(status, kStatusNonFinite);
    }
  }
  if (!write) return;
  uint4* dst = reinterpret_cast<uint4*>(out + (dst_row != nullptr ? dst_row[item] + j : row) * d + sub * 16);
  if (!real) {
    dst[0] = make_uint4(0, 0, 0, 0);
    dst[1] = make_uint4(0, 0, 0, 0);
    return;
  }
  const float inv = assume_normalized ? 1.0f : __fdiv_rn(1.0f, __fsqrt_rn(acc));
  uint32_t w[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const float a = assume_normalized ? x[2 * i] : __fmul_rn(x[2 * i], inv);
    const float b = assume_normalized ? x[2 * i + 1] : __fmul_rn(x[2 * i + 1], inv);
    w[i] = (uint32_t)__bfloat16_as_ushort(__float2bfloat16_rn(a)) |
           ((uint32_t)__bfloat16_as_ushort(__float2bfloat16_rn(b)) << 16);
  }
  dst[0] = make_uint4(w[0], w[1], w[2], w[3]);
  dst[1] = make_uint4(w[4], w[5], w[6], w[7]);
}

template <typename Tin, int TPR>
__global__ void __launch_bounds__(256) norm_layout_tpr_kernel(const Tin* in, int64_t n_src, int32_t in_rows,
                                                              const int32_t* __restrict__ lens,
                                                              int64_t n_items, int32_t out_rows, int32_t d,
                                                              uint32_t assume_normalized,
                                                              uint32_t check_finite,
                                                              __nv_bfloat16* out, uint32_t* status,
                                                              const int64_t* __restrict__ dst_row) {
  const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  norm_row_group<Tin, TPR>(tid / TPR, (uint32_t)(tid % TPR), in, n_src, in_rows, lens, n_items, out_rows,
                           d, assume_normalized, check_finite, out, status, dst_row);
}

// Packed layout (N4): the padding rows of chunk c's last 16-row group (rows len .. roundup(len,16)-1
// of its slot) become copies of its last real row.  The MaxSim kernel's packed epilogue then takes
// an unmasked max over every 16-column group: a repeated column cannot change a maximum, so the
// result is the max over the chunk's real columns exactly (reading R2), with no per-tail masking.
// Runs after the NORM launch (stream order), so it copies the final bf16 row.  One thread per
// (chunk, 16-byte word of a row).
__global__ void __launch_bounds__(256) pack_pad_replicate_kernel(__nv_bfloat16* tok,
                                                                 const int64_t* __restrict__ dst_row,
                                                                 const int32_t* __restrict__ lens,
                                                                 int64_t n, int32_t d) {
  const int32_t wpr = d / 8;  // uint4 words per row
  const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t c = tid / wpr;
  if (c >= n) return;
  const int32_t len = lens[c], end = (len + 15) & ~15;
  if (len == end) return;
  uint4* base = reinterpret_cast<uint4*>(tok + dst_row[c] * (int64_t)d) + (tid - c * wpr);
  const uint4 v = base[(int64_t)(len - 1) * wpr];
  for (int32_t j = len; j < end; ++j) base[(int64_t)j * wpr] = v;
}

// Two layouts in one launch (the ColTrast step: queries and documents): blocks [0, blocks_a) lay out
// segment A, the rest segment B.  Same per-row NORM as above.
struct NormSeg {
  const void* in;
  int64_t n_src;
  int32_t in_rows;
  const int32_t* lens;
  int64_t n_items;
  int32_t out_rows;
  __nv_bfloat16* out;
};
template <typename Tin, int TPR>
__global__ void __launch_bounds__(256) norm_layout2_kernel(NormSeg a, NormSeg b, int64_t blocks_a,
                                                           int32_t d, uint32_t assume_normalized,
                                                           uint32_t check_finite, uint32_t* status) {
  const bool first = (int64_t)blockIdx.x < blocks_a;
  const NormSeg& g = first ? a : b;
  const int64_t blk = first ? (int64_t)blockIdx.x : (int64_t)blockIdx.x - blocks_a;
  const int64_t tid = blk * blockDim.x + threadIdx.x;
  norm_row_group<Tin, TPR>(tid / TPR, (uint32_t)(tid % TPR), (const Tin*)g.in, g.n_src, g.in_rows,
                           g.lens, g.n_items, g.out_rows, d, assume_normalized, check_finite, g.out,
                           status, nullptr);
}

}  // namespace hiper
