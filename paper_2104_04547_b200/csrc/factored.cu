// Pocket-invariant factoring of the voxel head's first layer and the pocket
// cache helpers (fs_pocket_prepare / fs_score_poses_cached).
//
// conv1 is linear and the pocket and ligand channels are disjoint
// (channel = role*c_elem + element, complexes.py:182), so for a pose
//   conv1(grid) + b = [conv1(pocket channels) + b] + conv1(ligand channels).
// The bracket is computed once per pocket (fp32, cache); per pose only the
// ligand atoms are scattered through the 5^3 kernel.  Weights are the bf16
// values the tcgen05 conv1 uses, so the factored layer differs from the
// fused one only by fp32 summation order.  The output (ReLU, bf16,
// chunk-major [P][C/8][D][H][W][8]) feeds the tcgen05 conv2 unchanged.
#include <cuda_bf16.h>

#include "common.cuh"

namespace fs {

struct Conv1FactArgs {
  fs_pose_batch b;
  const char* cache; int64_t cache_stride; int64_t off_pp;   // pre-activation [G^3][COUT] fp32 per pocket
  const float* w;               // conv1 weights [k^3][cin][cout] fp32 (rounded to bf16 here)
  int c_elem; double box;
  __nv_bfloat16* out;           // [P][COUT/8][G^3][8]
};

constexpr int kC1G = 16, kC1K = 5, kC1R = 2, kC1Out = 32, kC1MaxLig = 128;

// 256 threads = the 16x16 (h, w) columns; each walks d = 0..15.
__global__ void __launch_bounds__(256) conv1_fact_kernel(Conv1FactArgs a) {
  extern __shared__ __align__(16) float wl[];           // [k^3][c_elem][32] ligand-channel weights
  __shared__ int4 atoms[kC1MaxLig];                      // (ix, iy, iz, ligand channel)
  const int p = blockIdx.x;
  const PoseView pv = pose_view(a.b, p);
  const int nL = (int)pv.na;
  if (nL > kC1MaxLig || pv.np_ == 0) return;             // not factorable (flagged by graph_fact_kernel)
  const int cin = 2 * a.c_elem;
  const int kk = kC1K * kC1K * kC1K;
  for (int i = threadIdx.x; i < kk * a.c_elem * kC1Out; i += blockDim.x) {
    const int o = i % kC1Out, c = (i / kC1Out) % a.c_elem, k = i / (kC1Out * a.c_elem);
    wl[i] = __bfloat162float(__float2bfloat16_rn(a.w[(static_cast<int64_t>(k) * cin + a.c_elem + c) * kC1Out + o]));
  }
  const double half = a.box / 2.0, gd = kC1G;
  for (int s = threadIdx.x; s < nL; s += blockDim.x) {
    double x, y, z; int32_t e, r;
    pv.atom(pv.np_ + s, x, y, z, e, r);
    // voxel index exactly as the voxelizer (complexes.py:180-181)
    auto ax = [&](double v) {
      double t = __dmul_rn(__ddiv_rn(__dadd_rn(v, half), a.box), gd);
      t = floor(t);
      t = fmin(fmax(t, 0.0), gd - 1.0);
      return (int)t;
    };
    atoms[s] = make_int4(ax(x), ax(y), ax(z), min(max(e, 0), a.c_elem - 1));
  }
  __syncthreads();
  const int h = threadIdx.x >> 4, w = threadIdx.x & 15;
  uint32_t near[kC1MaxLig / 32];
#pragma unroll
  for (int wd = 0; wd < kC1MaxLig / 32; ++wd) {
    uint32_t m = 0u;
    for (int s = 32 * wd; s < min(nL, 32 * wd + 32); ++s) {
      const int4 at = atoms[s];
      if (abs(at.y - h) <= kC1R && abs(at.z - w) <= kC1R) m |= 1u << (s & 31);
    }
    near[wd] = m;
  }
  const float* pp = reinterpret_cast<const float*>(a.cache + static_cast<int64_t>(a.b.pose_target[p]) * a.cache_stride +
                                                   a.off_pp);
  constexpr int64_t G3 = kC1G * kC1G * kC1G;
  for (int d = 0; d < kC1G; ++d) {
    const int vox = (d * kC1G + h) * kC1G + w;
    float acc[kC1Out];
    const float4* src = reinterpret_cast<const float4*>(pp + static_cast<int64_t>(vox) * kC1Out);
#pragma unroll
    for (int q = 0; q < kC1Out / 4; ++q) {
      const float4 v = __ldg(src + q);
      acc[4 * q] = v.x; acc[4 * q + 1] = v.y; acc[4 * q + 2] = v.z; acc[4 * q + 3] = v.w;
    }
    // ligand atoms in deterministic (atom) order: out[o] += W[v - o + r] (cross-correlation, 'same')
#pragma unroll
    for (int wd = 0; wd < kC1MaxLig / 32; ++wd) {
      uint32_t bits = near[wd];
      while (bits) {
        const int s = 32 * wd + __ffs(bits) - 1;
        bits &= bits - 1;
        const int4 at = atoms[s];
        const int kd = at.x - d + kC1R;
        if (kd < 0 || kd >= kC1K) continue;
        const int k = (kd * kC1K + (at.y - h + kC1R)) * kC1K + (at.z - w + kC1R);
        const float4* wk = reinterpret_cast<const float4*>(wl + (k * a.c_elem + at.w) * kC1Out);
#pragma unroll
        for (int q = 0; q < kC1Out / 4; ++q) {
          const float4 v = wk[q];
          acc[4 * q] += v.x; acc[4 * q + 1] += v.y; acc[4 * q + 2] += v.z; acc[4 * q + 3] += v.w;
        }
      }
    }
    uint4* op = reinterpret_cast<uint4*>(a.out) + static_cast<int64_t>(p) * (kC1Out / 8) * G3 + vox;
#pragma unroll
    for (int q = 0; q < kC1Out / 8; ++q) {
      uint4 pk;
      __nv_bfloat162* b2 = reinterpret_cast<__nv_bfloat162*>(&pk);
#pragma unroll
      for (int t = 0; t < 4; ++t)
        b2[t] = __floats2bfloat162_rn(fmaxf(acc[8 * q + 2 * t], 0.f), fmaxf(acc[8 * q + 2 * t + 1], 0.f));
      op[q * G3] = pk;
    }
  }
}

bool conv1_fact_supported(int g, int k, int cin, int cout) {
  return g == kC1G && k == kC1K && cout == kC1Out && cin % 2 == 0 && cin / 2 <= 8;
}

int launch_conv1_fact(const fs_pose_batch& b, const char* cache, int64_t cache_stride, int64_t off_pp, const float* w,
                      int c_elem, double box, __nv_bfloat16* out, cudaStream_t st) {
  if (b.n_poses <= 0) return FS_OK;
  Conv1FactArgs a;
  a.b = b; a.cache = cache; a.cache_stride = cache_stride; a.off_pp = off_pp; a.w = w;
  a.c_elem = c_elem; a.box = box; a.out = out;
  const size_t smem = static_cast<size_t>(kC1K * kC1K * kC1K) * c_elem * kC1Out * 4;
  FS_CUDA_CHECK(cudaFuncSetAttribute(conv1_fact_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  conv1_fact_kernel<<<b.n_poses, 256, smem, st>>>(a);
  FS_LAUNCH_CHECK();
  return FS_OK;
}

// ---- pocket preparation helpers ---------------------------------------------
// weights rounded to the bf16 values of the tensor-core conv1
__global__ void round_bf16_kernel(const float* in, float* out, int64_t n) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) out[i] = __bfloat162float(__float2bfloat16_rn(in[i]));
}

int launch_round_bf16(const float* in, float* out, int64_t n, cudaStream_t st) {
  if (n <= 0) return FS_OK;
  round_bf16_kernel<<<(unsigned)cdiv(n, 256), 256, 0, st>>>(in, out, n);
  FS_LAUNCH_CHECK();
  return FS_OK;
}

// T[c] = sum over the pocket's nodes of f[node][c] (float64, node order)
__global__ void pocket_total_kernel(const int64_t* pocket_off, const float* f, int64_t ld, char* cache,
                                    int64_t cache_stride, int64_t off_T, int64_t off_n) {
  const int q = blockIdx.x;
  const int n = static_cast<int>(pocket_off[q + 1] - pocket_off[q]);
  char* c = cache + static_cast<int64_t>(q) * cache_stride;
  if (threadIdx.x < 128) {
    double t = 0.0;
    const float* fq = f + static_cast<int64_t>(q) * ld * 128;
    for (int i = 0; i < n; ++i) t += static_cast<double>(fq[static_cast<int64_t>(i) * 128 + threadIdx.x]);
    reinterpret_cast<double*>(c + off_T)[threadIdx.x] = t;
  }
  if (threadIdx.x == 0) *reinterpret_cast<int32_t*>(c + off_n) = n;
}

int launch_pocket_total(const int64_t* pocket_off, int n_pockets, const float* f, int64_t ld, char* cache,
                        int64_t cache_stride, int64_t off_T, int64_t off_n, cudaStream_t st) {
  if (n_pockets <= 0) return FS_OK;
  pocket_total_kernel<<<n_pockets, 128, 0, st>>>(pocket_off, f, ld, cache, cache_stride, off_T, off_n);
  FS_LAUNCH_CHECK();
  return FS_OK;
}

// pocket-only pose batch: pose q = pocket q with no ligand atoms
__global__ void pocket_poses_kernel(int n, int64_t* atom_off, int32_t* target) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i <= n) atom_off[i] = 0;
  if (i < n) target[i] = i;
}

int launch_pocket_poses(int n, int64_t* atom_off, int32_t* target, cudaStream_t st) {
  pocket_poses_kernel<<<(unsigned)cdiv(n + 1, 256), 256, 0, st>>>(n, atom_off, target);
  FS_LAUNCH_CHECK();
  return FS_OK;
}

}  // namespace fs
