// Ranking kernels: top-k merge and per-compound best pose.
//
// Tie rule of evaluate.aggregate_best_pose (evaluate.py:67-83): higher score
// first, ties to the lowest pose id.  The reference has no top-k; ranking the
// whole library by (score desc, global pose index asc) is the natural
// extension the multi-GPU merge needs.
#include <cub/cub.cuh>

#include "common.cuh"

namespace fs {

// Monotone map: ascending key <=> (score descending); NaN last; -0 == +0.
__device__ __forceinline__ uint32_t score_desc_bits(float s) {
  if (isnan(s)) return 0xffffffffu;
  if (s == 0.0f) s = 0.0f;
  uint32_t u = __float_as_uint(s);
  u = (u & 0x80000000u) ? ~u : (u | 0x80000000u);   // ascending float order
  return ~u;                                         // descending
}

__device__ __forceinline__ float score_from_bits(uint32_t k) {
  if (k == 0xffffffffu) return __int_as_float(0x7fc00000);
  uint32_t u = ~k;
  u = (u & 0x80000000u) ? (u & 0x7fffffffu) : ~u;
  return __uint_as_float(u);
}

// Two stable radix passes give the order (score desc, index asc) over the full
// 64-bit pose index: sort by index, then stably by the 32-bit score key.
__device__ __forceinline__ uint64_t index_key(int64_t i) {   // signed -> unsigned order
  return static_cast<uint64_t>(i) ^ 0x8000000000000000ull;
}

__global__ void topk_keys_kernel(const float* as, const int64_t* ai, int64_t na, const float* bs,
                                 const int64_t* bi, int64_t nb, uint64_t* idx_keys, uint32_t* score_keys) {
  int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= na + nb) return;
  float s; int64_t i;
  if (t < na) { s = as[t]; i = ai[t]; } else { s = bs[t - na]; i = bi[t - na]; }
  idx_keys[t] = index_key(i);
  score_keys[t] = score_desc_bits(s);
}

__global__ void topk_decode_kernel(const uint32_t* score_keys, const uint64_t* idx_keys, int64_t k, float* os,
                                   int64_t* oi) {
  int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= k) return;
  os[t] = score_from_bits(score_keys[t]);
  oi[t] = static_cast<int64_t>(idx_keys[t] ^ 0x8000000000000000ull);
}

static size_t topk_tmp_bytes(int64_t n) {
  size_t t1 = 0, t2 = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, t1, (uint64_t*)nullptr, (uint64_t*)nullptr, (uint32_t*)nullptr,
                                  (uint32_t*)nullptr, (int)n);
  cub::DeviceRadixSort::SortPairs(nullptr, t2, (uint32_t*)nullptr, (uint32_t*)nullptr, (uint64_t*)nullptr,
                                  (uint64_t*)nullptr, (int)n);
  return t1 > t2 ? t1 : t2;
}

size_t topk_ws_bytes(int64_t n) { return topk_tmp_bytes(n) + 2 * (size_t)n * (8 + 4) + 1024; }

int launch_topk_merge(const float* as, const int64_t* ai, int64_t na, const float* bs,
                      const int64_t* bi, int64_t nb, int k, float* os, int64_t* oi, void* ws,
                      size_t ws_bytes, cudaStream_t st) {
  const int64_t n = na + nb;
  if (k < 0) return FS_EINVAL;
  if (n == 0 || k == 0) return FS_OK;
  if ((size_t)topk_ws_bytes(n) > ws_bytes) return FS_ECAPACITY;
  uint64_t* ik0 = (uint64_t*)ws;
  uint64_t* ik1 = ik0 + n;
  uint32_t* sk0 = (uint32_t*)(ik1 + n);
  uint32_t* sk1 = sk0 + n;
  void* tmp = (void*)(((uintptr_t)(sk1 + n) + 255) & ~(uintptr_t)255);
  size_t tmp_bytes = topk_tmp_bytes(n);
  topk_keys_kernel<<<(unsigned)cdiv(n, 256), 256, 0, st>>>(as, ai, na, bs, bi, nb, ik0, sk0);
  FS_LAUNCH_CHECK();
  // pass 1: by pose index (all 64 bits); pass 2: stably by score key
  FS_CUDA_CHECK(cub::DeviceRadixSort::SortPairs(tmp, tmp_bytes, ik0, ik1, sk0, sk1, (int)n, 0, 64, st));
  FS_CUDA_CHECK(cub::DeviceRadixSort::SortPairs(tmp, tmp_bytes, sk1, sk0, ik1, ik0, (int)n, 0, 32, st));
  const int64_t kk = k < n ? k : n;
  topk_decode_kernel<<<(unsigned)cdiv(kk, 256), 256, 0, st>>>(sk0, ik0, kk, os, oi);
  FS_LAUNCH_CHECK();
  return FS_OK;
}

// best pose per compound: key = (score-order bits, pose id) min-reduced.
__global__ void best_key_kernel(const int64_t* compound, const int64_t* pose_id, const float* s,
                                int64_t n, int dir, unsigned long long* best) {
  int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n) return;
  float v = dir > 0 ? s[t] : -s[t];
  unsigned long long key = ((unsigned long long)score_desc_bits(v) << 32) | (uint32_t)pose_id[t];
  atomicMin(&best[compound[t]], key);
}

__global__ void best_idx_kernel(const int64_t* compound, const int64_t* pose_id, const float* s,
                                int64_t n, int dir, const unsigned long long* best, int64_t* idx) {
  int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n) return;
  float v = dir > 0 ? s[t] : -s[t];
  unsigned long long key = ((unsigned long long)score_desc_bits(v) << 32) | (uint32_t)pose_id[t];
  if (key == best[compound[t]]) atomicMin((unsigned long long*)&idx[compound[t]], (unsigned long long)t);
}

int launch_best_pose(const int64_t* compound, const int64_t* pose_id, const float* s, int64_t n,
                     int64_t n_compounds, int dir, int64_t* best_idx, uint64_t* best_key,
                     cudaStream_t st) {
  if (dir != 1 && dir != -1) return FS_EINVAL;
  if (n_compounds <= 0) return FS_OK;
  // all-ones: the unsigned atomicMin sentinel, and -1 (no rows) as int64
  FS_CUDA_CHECK(cudaMemsetAsync(best_idx, 0xff, sizeof(int64_t) * n_compounds, st));
  unsigned long long* keys = (unsigned long long*)best_key;
  FS_CUDA_CHECK(cudaMemsetAsync(keys, 0xff, sizeof(unsigned long long) * n_compounds, st));
  best_key_kernel<<<(unsigned)cdiv(n, 256), 256, 0, st>>>(compound, pose_id, s, n, dir, keys);
  FS_LAUNCH_CHECK();
  best_idx_kernel<<<(unsigned)cdiv(n, 256), 256, 0, st>>>(compound, pose_id, s, n, dir, keys, best_idx);
  FS_LAUNCH_CHECK();
  return FS_OK;
}

// Streaming form: fold a batch into per-compound keys (no reset), then decode.
__global__ void best_update_kernel(const int64_t* compound, int64_t base, const int64_t* pose_id, const float* s,
                                   int64_t n, int64_t n_compounds, int dir, unsigned long long* best) {
  int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n) return;
  const int64_t c = compound[t] - base;
  if (c < 0 || c >= n_compounds) return;
  float v = dir > 0 ? s[t] : -s[t];
  unsigned long long key = ((unsigned long long)score_desc_bits(v) << 32) | (uint32_t)pose_id[t];
  atomicMin(&best[c], key);
}

__global__ void best_decode_kernel(const unsigned long long* best, int64_t n, int dir, float* score,
                                   int64_t* pose) {
  int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n) return;
  const unsigned long long k = best[t];
  if (k == ~0ull) { score[t] = __int_as_float(0x7fc00000); pose[t] = -1; return; }
  const float v = score_from_bits((uint32_t)(k >> 32));
  score[t] = dir > 0 ? v : -v;
  pose[t] = (int64_t)(uint32_t)k;
}

int launch_best_update(const int64_t* compound, int64_t base, const int64_t* pose_id, const float* s, int64_t n,
                       int64_t n_compounds, int dir, uint64_t* best_key, cudaStream_t st) {
  if (dir != 1 && dir != -1) return FS_EINVAL;
  if (n <= 0) return FS_OK;
  best_update_kernel<<<(unsigned)cdiv(n, 256), 256, 0, st>>>(compound, base, pose_id, s, n, n_compounds, dir,
                                                            (unsigned long long*)best_key);
  FS_LAUNCH_CHECK();
  return FS_OK;
}

int launch_best_decode(const uint64_t* best_key, int64_t n, int dir, float* score, int64_t* pose, cudaStream_t st) {
  if (dir != 1 && dir != -1) return FS_EINVAL;
  if (n <= 0) return FS_OK;
  best_decode_kernel<<<(unsigned)cdiv(n, 256), 256, 0, st>>>((const unsigned long long*)best_key, n, dir, score, pose);
  FS_LAUNCH_CHECK();
  return FS_OK;
}

}  // namespace fs
