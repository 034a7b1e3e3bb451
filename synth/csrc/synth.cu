// synth.cu -- device implementation of synth/gen.py's counter-based generator (same integer recipe,
// bit-identical outputs; checked by tests/test_gpu_parity.py::test_synth_device_matches_numpy).  Holds none of the method's arithmetic:
// it only draws raw token embeddings for benchmarks/tests at sizes numpy cannot produce quickly
// (e.g. a 1M x 256 x 128 corpus, 65.5 GB, generated directly in HBM).
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <cstdint>

namespace {

enum { TOK = 1, CENT = 2, TOPIC = 3, TOPIC2 = 4, MIX = 5, LEN = 6, QTARGET = 7, QPOS = 8, QTOK = 9 };
constexpr uint64_t kTopics = 4096;

__host__ __device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  uint64_t z = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
__host__ __device__ __forceinline__ uint64_t key_of(uint64_t seed, uint64_t stream) {
  return splitmix64(seed ^ (stream << 48));
}
__device__ __forceinline__ float g_of(uint64_t h) {
  const int64_t s = (int64_t)((h & 0xFFFF) + ((h >> 16) & 0xFFFF) + ((h >> 32) & 0xFFFF) + (h >> 48)) - 131070;
  return __fmul_rn((float)s, 3.0517578125e-05f);  // 2^-15, exact
}
__device__ __forceinline__ uint16_t f2bf(float f) {
  return __bfloat16_as_ushort(__float2bfloat16_rn(f));
}

struct Keys {
  uint64_t tok, cent, topic, topic2, mix;
};

__device__ __forceinline__ float corpus_value(const Keys& K, int planted, uint64_t c, uint64_t j,
                                              uint64_t k, uint64_t L, uint64_t d, float sigma) {
  const float noise = g_of(splitmix64(K.tok + (c * L + j) * d + k));
  if (!planted) return noise;
  uint64_t t = splitmix64(K.topic + c) % kTopics;
  if ((splitmix64(K.mix + c * L + j) & 3ull) == 0) t = splitmix64(K.topic2 + c) % kTopics;
  const float cent = g_of(splitmix64(K.cent + t * d + k));
  return __fadd_rn(cent, __fmul_rn(sigma, noise));
}

__global__ void corpus_kernel(void* out, int out_bf16, uint64_t c0, uint64_t n, uint64_t L, uint64_t d,
                              Keys K, int planted, float sigma) {
  const uint64_t total = n * L * d;
  for (uint64_t e = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total;
       e += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t k = e % d;
    const uint64_t row = e / d;
    const uint64_t j = row % L;
    const uint64_t c = c0 + row / L;
    const float v = corpus_value(K, planted, c, j, k, L, d, sigma);
    if (out_bf16) reinterpret_cast<uint16_t*>(out)[e] = f2bf(v);
    else reinterpret_cast<float*>(out)[e] = v;
  }
}

// Queries: token i of query q copies corpus token (tgt(q), j) and adds sigma_q * g (planted);
// tgt/pos computed on device from the same hashes as gen.py.  chunk_lens (device, may be null =
// all L) gives len(tgt) for j = h(QPOS) % len.
__global__ void query_kernel(void* out, int out_bf16, uint64_t q0, uint64_t n_q, uint64_t Lq,
                             uint64_t d, uint64_t qtok, uint64_t qtarget, uint64_t qpos, int diagonal,
                             int query_planted, uint64_t n_chunks, uint64_t L, const int32_t* chunk_lens,
                             Keys K, int corpus_planted, float sigma, float sigma_q) {
  const uint64_t total = n_q * Lq * d;
  for (uint64_t e = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total;
       e += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t k = e % d;
    const uint64_t row = e / d;
    const uint64_t i = row % Lq;
    const uint64_t q = q0 + row / Lq;
    const float noise = g_of(splitmix64(qtok + (q * Lq + i) * d + k));
    float v = noise;
    if (query_planted) {
      const uint64_t tgt = diagonal ? (q % n_chunks) : (splitmix64(qtarget + q) % n_chunks);
      const uint64_t tl = chunk_lens ? (uint64_t)chunk_lens[tgt] : L;
      const uint64_t j = splitmix64(qpos + q * Lq + i) % tl;
      const float base = corpus_value(K, corpus_planted, tgt, j, k, L, d, sigma);
      v = __fadd_rn(base, __fmul_rn(sigma_q, noise));
    }
    if (out_bf16) reinterpret_cast<uint16_t*>(out)[e] = f2bf(v);
    else reinterpret_cast<float*>(out)[e] = v;
  }
}

// Corpus chunks written straight into a packed layout: chunk c's token j (< len[c]) goes to row
// dst_row[c] + j of out [rows][d] (bf16); rows len[c] .. roundup(len[c], 16) - 1 are zeroed.  The
// values are those of corpus_kernel for the same (chunk, token, dim) (L = the hash's token stride).
__global__ void corpus_packed_kernel(uint16_t* out, uint64_t c0, uint64_t n, uint64_t L, uint64_t d,
                                     const int64_t* dst_row, const int32_t* lens, Keys K, int planted,
                                     float sigma) {
  const uint64_t total = n * L * d;
  for (uint64_t e = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total;
       e += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t k = e % d;
    const uint64_t row = e / d;
    const uint64_t j = row % L;
    const uint64_t c = row / L;
    const uint64_t len = (uint64_t)lens[c];
    if (j >= ((len + 15) & ~15ull)) continue;
    const float v = j < len ? corpus_value(K, planted, c0 + c, j, k, L, d, sigma) : 0.0f;
    out[((uint64_t)dst_row[c] + j) * d + k] = f2bf(v);
  }
}

Keys make_keys(uint64_t seed) {
  return Keys{key_of(seed, TOK), key_of(seed, CENT), key_of(seed, TOPIC), key_of(seed, TOPIC2),
              key_of(seed, MIX)};
}

int grid_for(uint64_t total) {
  uint64_t b = (total + 255) / 256;
  return (int)(b > 148ull * 64 ? 148ull * 64 : (b ? b : 1));
}

}  // namespace

extern "C" __attribute__((visibility("default"))) int synth_corpus(void* out, int out_bf16, int64_t chunk_start, int64_t n, int32_t L,
                            int32_t d, uint64_t seed, int planted, float sigma, void* stream) {
  if (n <= 0) return 0;
  const uint64_t total = (uint64_t)n * L * d;
  corpus_kernel<<<grid_for(total), 256, 0, (cudaStream_t)stream>>>(
      out, out_bf16, (uint64_t)chunk_start, (uint64_t)n, (uint64_t)L, (uint64_t)d, make_keys(seed),
      planted, sigma);
  return (int)cudaGetLastError();
}

extern "C" __attribute__((visibility("default"))) int synth_queries(void* out, int out_bf16, int64_t q_start, int64_t n_q, int32_t Lq,
                             int32_t d, uint64_t qseed, int diagonal, int query_planted,
                             int64_t n_chunks, int32_t L, const int32_t* chunk_lens_dev,
                             uint64_t corpus_seed, int corpus_planted, float sigma, float sigma_q,
                             void* stream) {
  if (n_q <= 0) return 0;
  const uint64_t total = (uint64_t)n_q * Lq * d;
  query_kernel<<<grid_for(total), 256, 0, (cudaStream_t)stream>>>(
      out, out_bf16, (uint64_t)q_start, (uint64_t)n_q, (uint64_t)Lq, (uint64_t)d,
      key_of(qseed, QTOK), key_of(qseed, QTARGET), key_of(qseed, QPOS), diagonal, query_planted,
      (uint64_t)n_chunks, (uint64_t)L, chunk_lens_dev, make_keys(corpus_seed), corpus_planted, sigma,
      sigma_q);
  return (int)cudaGetLastError();
}

extern "C" __attribute__((visibility("default"))) int synth_corpus_packed(
    void* out, int64_t chunk_start, int64_t n, int32_t L, int32_t d, uint64_t seed, int planted,
    float sigma, const int64_t* dst_row_dev, const int32_t* lens_dev, void* stream) {
  if (n <= 0) return 0;
  const uint64_t total = (uint64_t)n * L * d;
  corpus_packed_kernel<<<grid_for(total), 256, 0, (cudaStream_t)stream>>>(
      (uint16_t*)out, (uint64_t)chunk_start, (uint64_t)n, (uint64_t)L, (uint64_t)d, dst_row_dev,
      lens_dev, make_keys(seed), planted, sigma);
  return (int)cudaGetLastError();
}
