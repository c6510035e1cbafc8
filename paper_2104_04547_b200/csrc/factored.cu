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

#include <algorithm>

#include "common.cuh"

namespace fs {

struct Conv1FactArgs {
  fs_pose_batch b;
  const char* cache; int64_t cache_stride;
  int64_t off_pp;               // pre-activation [G^3][COUT] fp32 (pocket channels + bias)
  int64_t off_ppact;            // relu(pre-activation) as bf16 in the act1 layout [COUT/8][G^3][8]
  int64_t off_wl;               // ligand-channel weights [k^3][c_elem][COUT], bf16-valued fp32
                                //   (X3 caches: the exact fp32 weights)
  int64_t off_ppact_lo;         // X3: the lo part of relu(pre-activation)
  int c_elem; double box;
  __nv_bfloat16* out;           // [P][COUT/8][G^3][8]
  __nv_bfloat16* out_lo;        // X3 (FS_PREC_MIXED): lo part, same layout
};

constexpr int kC1G = 16, kC1K = 5, kC1R = 2, kC1Out = 32, kC1MaxLig = 128;
constexpr int kC1G3 = kC1G * kC1G * kC1G;
constexpr int kC1Threads = 256;

// Persistent CTAs, one pose at a time:
//  1. ligand atoms -> voxels; mark every output voxel within the 5^3 window
//     of a ligand atom (bitmask);
//  2. voxels no ligand atom reaches: act1 = cached relu(pocket pre-activation)
//     (a 16-byte copy per 8 channels, L2 -> HBM);
//  3. reached voxels: pocket pre-activation + the ligand atoms' weights, in
//     atom order (deterministic), ReLU, bf16.
// X3: the layer in fp32 (exact weights) with the output as a (hi, lo) bf16 pair
// for the 3-pass tcgen05 conv2 (FS_PREC_MIXED)
template <bool X3>
__global__ void __launch_bounds__(kC1Threads) conv1_fact_kernel(Conv1FactArgs a) {
  extern __shared__ __align__(16) float wl[];           // [k^3][c_elem][32]
  __shared__ int4 atoms[kC1MaxLig];                      // (ix, iy, iz, ligand channel)
  __shared__ uint32_t near_hw[kC1G * kC1G][kC1MaxLig / 32];   // atoms whose 5x5 (h, w) window covers the column
  __shared__ uint32_t near_d[kC1G][kC1MaxLig / 32];            // atoms whose 5-plane d window covers the plane
  __shared__ uint32_t touched[kC1G3 / 32];
  __shared__ int s_cnt;
  __shared__ uint16_t tlist[kC1G3];
  const int nw = kC1K * kC1K * kC1K * a.c_elem * kC1Out;
  const char* c0 = a.cache;   // the weights are identical in every pocket slot
  // weight row R (32 floats = 8 float4) is stored with its float4 q at slot
  // (q + R) & 7: the lanes of a warp read different rows, which would all
  // hit the same 4 banks unswizzled (128-byte row stride)
  for (int i = threadIdx.x; i < nw / 4; i += blockDim.x) {
    const int row = i >> 3, q = i & 7;
    reinterpret_cast<float4*>(wl)[row * 8 + ((q + row) & 7)] = reinterpret_cast<const float4*>(c0 + a.off_wl)[i];
  }
  const double half = a.box / 2.0, gd = kC1G;
  for (int p = blockIdx.x; p < a.b.n_poses; p += gridDim.x) {
    const PoseView pv = pose_view(a.b, p);
    const int nL = (int)pv.na;
    if (nL > kC1MaxLig || pv.np_ == 0) continue;         // not factorable (flagged by graph_fact_kernel)
    __syncthreads();                                     // previous pose done with atoms/touched/tlist
    for (int i = threadIdx.x; i < kC1G * kC1G * (kC1MaxLig / 32); i += blockDim.x) (&near_hw[0][0])[i] = 0u;
    for (int i = threadIdx.x; i < kC1G * (kC1MaxLig / 32); i += blockDim.x) (&near_d[0][0])[i] = 0u;
    if (threadIdx.x == 0) s_cnt = 0;
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
    for (int i = threadIdx.x; i < nL * 30; i += blockDim.x) {
      const int sidx = i / 30, k = i % 30;
      const int4 at = atoms[sidx];
      const uint32_t bit = 1u << (sidx & 31);
      if (k < 25) {
        const int h = at.y + k / 5 - kC1R, w = at.z + k % 5 - kC1R;
        if (h >= 0 && h < kC1G && w >= 0 && w < kC1G) atomicOr(&near_hw[h * kC1G + w][sidx >> 5], bit);
      } else {
        const int d = at.x + (k - 25) - kC1R;
        if (d >= 0 && d < kC1G) atomicOr(&near_d[d][sidx >> 5], bit);
      }
    }
    __syncthreads();
    const char* pc = a.cache + static_cast<int64_t>(a.b.pose_target[p]) * a.cache_stride;
    const uint4* ppact = reinterpret_cast<const uint4*>(pc + a.off_ppact);
    const uint4* ppact_lo = reinterpret_cast<const uint4*>(pc + a.off_ppact_lo);
    uint4* op = reinterpret_cast<uint4*>(a.out) + static_cast<int64_t>(p) * (kC1Out / 8) * kC1G3;
    uint4* op_lo = X3 ? reinterpret_cast<uint4*>(a.out_lo) + static_cast<int64_t>(p) * (kC1Out / 8) * kC1G3 : nullptr;
    // untouched voxels: copy; touched ones: list them
    // touched-voxel bitmask, then the copy of the untouched ones with 4
    // independent 16-byte loads in flight per thread
    for (int vw = threadIdx.x; vw < kC1G3 / 32; vw += blockDim.x) {
      uint32_t m = 0u;
      for (int b = 0; b < 32; ++b) {
        const int v = 32 * vw + b;
        uint32_t any = 0u;
#pragma unroll
        for (int wd = 0; wd < kC1MaxLig / 32; ++wd) any |= near_hw[v & 255][wd] & near_d[v >> 8][wd];
        m |= (any ? 1u : 0u) << b;
      }
      touched[vw] = m;
    }
    __syncthreads();
    constexpr int kUnits = (kC1Out / 8) * kC1G3;
    for (int u0 = threadIdx.x; u0 < kUnits; u0 += 4 * kC1Threads) {
      uint4 x[4];
      bool t[4];
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        const int u = u0 + r * kC1Threads;
        const int v = u & (kC1G3 - 1);
        t[r] = u >= kUnits || ((touched[v >> 5] >> (v & 31)) & 1u);
        if (!t[r]) x[r] = __ldg(ppact + u);
      }
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        const int u = u0 + r * kC1Threads;
        if (u >= kUnits) continue;
        if (!t[r]) {
          op[u] = x[r];
          if constexpr (X3) op_lo[u] = __ldg(ppact_lo + u);
        } else if (u < kC1G3) {
          tlist[atomicAdd(&s_cnt, 1)] = static_cast<uint16_t>(u);
        }
      }
    }
    __syncthreads();
    const float* pp = reinterpret_cast<const float*>(pc + a.off_pp);
    const int nt = s_cnt;
    for (int i = threadIdx.x; i < nt; i += blockDim.x) {
      const int v = tlist[i];
      const int d = v >> 8, h = (v >> 4) & 15, w = v & 15;
      float acc[kC1Out];
      const float4* src = reinterpret_cast<const float4*>(pp + static_cast<int64_t>(v) * kC1Out);
#pragma unroll
      for (int q = 0; q < kC1Out / 4; ++q) {
        const float4 x = __ldg(src + q);
        acc[4 * q] = x.x; acc[4 * q + 1] = x.y; acc[4 * q + 2] = x.z; acc[4 * q + 3] = x.w;
      }
      // out[o] += W[v_atom - o + r] (cross-correlation, 'same'), in atom
      // order over exactly the atoms whose window covers this voxel
#pragma unroll
      for (int wd = 0; wd < kC1MaxLig / 32; ++wd) {
        uint32_t bits = near_hw[v & 255][wd] & near_d[d][wd];
        while (bits) {
          const int sidx = 32 * wd + __ffs(bits) - 1;
          bits &= bits - 1;
          const int4 at = atoms[sidx];
          const int k = ((at.x - d + kC1R) * kC1K + (at.y - h + kC1R)) * kC1K + (at.z - w + kC1R);
          const int row = k * a.c_elem + at.w;
          const float4* wk = reinterpret_cast<const float4*>(wl) + row * 8;
#pragma unroll
          for (int q = 0; q < kC1Out / 4; ++q) {
            const float4 x = wk[(q + row) & 7];
            acc[4 * q] += x.x; acc[4 * q + 1] += x.y; acc[4 * q + 2] += x.z; acc[4 * q + 3] += x.w;
          }
        }
      }
#pragma unroll
      for (int q = 0; q < kC1Out / 8; ++q) {
        uint4 pk, pl;
        __nv_bfloat162* b2 = reinterpret_cast<__nv_bfloat162*>(&pk);
        __nv_bfloat162* l2 = reinterpret_cast<__nv_bfloat162*>(&pl);
#pragma unroll
        for (int t = 0; t < 4; ++t) {
          const float x0 = fmaxf(acc[8 * q + 2 * t], 0.f), x1 = fmaxf(acc[8 * q + 2 * t + 1], 0.f);
          b2[t] = __floats2bfloat162_rn(x0, x1);
          if constexpr (X3) {
            const float2 h = __bfloat1622float2(b2[t]);
            l2[t] = __floats2bfloat162_rn(x0 - h.x, x1 - h.y);
          }
        }
        op[q * kC1G3 + v] = pk;
        if constexpr (X3) op_lo[q * kC1G3 + v] = pl;
      }
    }
  }
}

bool conv1_fact_supported(int g, int k, int cin, int cout) {
  return g == kC1G && k == kC1K && cout == kC1Out && cin % 2 == 0 && cin / 2 <= 8;
}

template <bool X3>
static int launch_conv1_fact_t(const Conv1FactArgs& a, int n_poses, size_t smem, cudaStream_t st) {
  FS_CUDA_CHECK(cudaFuncSetAttribute(conv1_fact_kernel<X3>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int dev = 0, sms = 148, per_sm = 1;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, conv1_fact_kernel<X3>, kC1Threads, smem);
  const int grid = static_cast<int>(std::min<int64_t>(n_poses, static_cast<int64_t>(sms) * std::max(per_sm, 1)));
  conv1_fact_kernel<X3><<<grid, kC1Threads, smem, st>>>(a);
  FS_LAUNCH_CHECK();
  return FS_OK;
}

int launch_conv1_fact(const fs_pose_batch& b, const char* cache, int64_t cache_stride, int64_t off_pp,
                      int64_t off_ppact, int64_t off_wl, int c_elem, double box, __nv_bfloat16* out, cudaStream_t st,
                      int64_t off_ppact_lo, __nv_bfloat16* out_lo) {
  if (b.n_poses <= 0) return FS_OK;
  Conv1FactArgs a;
  a.b = b; a.cache = cache; a.cache_stride = cache_stride; a.off_pp = off_pp; a.off_ppact = off_ppact;
  a.off_wl = off_wl; a.c_elem = c_elem; a.box = box; a.out = out;
  a.off_ppact_lo = off_ppact_lo; a.out_lo = out_lo;
  const size_t smem = static_cast<size_t>(kC1K * kC1K * kC1K) * c_elem * kC1Out * 4;
  return out_lo ? launch_conv1_fact_t<true>(a, b.n_poses, smem, st) : launch_conv1_fact_t<false>(a, b.n_poses, smem, st);
}

// cache fields derived from the pocket pre-activation: relu'd bf16 act1
// layout, and (slot-independent) the ligand-channel weights as bf16 values
// x3 (FS_PREC_MIXED caches): relu'd act1 as a (hi, lo) pair and the exact fp32
// ligand-channel weights
__global__ void pocket_conv1_fields_kernel(const float* pp, int64_t pp_ld, char* cache, int64_t cache_stride,
                                           int64_t off_ppact, int64_t off_wl, const float* w1, int c_elem,
                                           int64_t off_ppact_lo, int x3) {
  const int q = blockIdx.y;
  const float* src = pp + static_cast<int64_t>(q) * pp_ld;
  char* c = cache + static_cast<int64_t>(q) * cache_stride;
  __nv_bfloat16* act = reinterpret_cast<__nv_bfloat16*>(c + off_ppact);
  __nv_bfloat16* act_lo = reinterpret_cast<__nv_bfloat16*>(c + off_ppact_lo);
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < kC1G3 * kC1Out; i += gridDim.x * blockDim.x) {
    const int v = i / kC1Out, o = i % kC1Out;
    const float x = fmaxf(src[i], 0.f);
    const __nv_bfloat16 h = __float2bfloat16_rn(x);
    const int64_t at = (static_cast<int64_t>(o / 8) * kC1G3 + v) * 8 + (o & 7);
    act[at] = h;
    if (x3) act_lo[at] = __float2bfloat16_rn(x - __bfloat162float(h));
  }
  float* wlc = reinterpret_cast<float*>(c + off_wl);
  const int cin = 2 * c_elem, nw = kC1K * kC1K * kC1K * c_elem * kC1Out;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < nw; i += gridDim.x * blockDim.x) {
    const int o = i % kC1Out, ch = (i / kC1Out) % c_elem, k = i / (kC1Out * c_elem);
    const float wv = w1[(static_cast<int64_t>(k) * cin + c_elem + ch) * kC1Out + o];
    wlc[i] = x3 ? wv : __bfloat162float(__float2bfloat16_rn(wv));
  }
}

int launch_pocket_conv1_fields(const float* pp, int n_pockets, char* cache, int64_t cache_stride, int64_t off_ppact,
                               int64_t off_wl, const float* w1, int c_elem, cudaStream_t st, int64_t off_ppact_lo,
                               int x3) {
  if (n_pockets <= 0) return FS_OK;
  dim3 grid(64, n_pockets);
  pocket_conv1_fields_kernel<<<grid, 256, 0, st>>>(pp, static_cast<int64_t>(kC1G3) * kC1Out, cache, cache_stride,
                                                   off_ppact, off_wl, w1, c_elem, off_ppact_lo, x3);
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
