// SG-CNN head: gated (GRU-style) message passing + gated gather + per-pose
// mean pool, fused into one kernel per pose (fp32, deterministic).
//
// Reference: _graph_tape / _gru_phase (models.py:334-371), neighbor-sum
// (autodiff.py:527-539), pool matrix rows 1/n (models.py:249-254).
//   per step: m = A.(h.W_msg); z = s(m.Wz+bz+h.Uz); r = s(m.Wr+br+h.Ur);
//             hh = tanh(m.Wh+bh+(r*h).Uh); h <- h + z*(hh-h)
// We use the exact real-arithmetic identity m.Wg = (A.h).(W_msg.Wg): the
// host folds W_msg into the three gate matrices (fp64), so each step is one
// neighbour SUM of h rows and three small fused GEMVs per node.
// Determinism: every node row is summed in CSR order (ascending neighbour
// id) by one thread; pooling uses a fixed per-thread node assignment and a
// fixed shuffle tree.  Hence a pose's output is bitwise independent of the
// batch it is scored in (SPEC.md:275 asks 1e-10).
#include "common.cuh"

namespace fs {

struct GnnArgs {
  const float* feats; int F;            // [N][F]
  const int64_t* node_off;
  const int64_t* row_cov; const int32_t* deg_cov; const col_t* col_cov;     // row start + degree
  const int64_t* row_ncov; const int32_t* deg_ncov; const col_t* col_ncov;
  const float* we; const float* be;     // [F][D], [D]
  const float* phase[2];                // per phase: Wc[D][3D] | bc[3D] | U[D][2D] | Uh[D][D]
  const float* gg; const float* bg;     // [D][GN], [GN]
  const float* gf; const float* bf;
  int k_steps[2]; int gn;
  float* state;                         // global fallback [2][N][D] (nullable)
  float* lat; int64_t ld_lat;           // [P][ld_lat], columns 0..GN-1
  const int32_t* err;
  int smem_state;                       // 1: node state in shared memory
};

template <int D>
__host__ __device__ constexpr int phase_floats() { return D * 3 * D + 3 * D + D * 2 * D + D * D; }

constexpr int kGnnThreads = 384;

template <int D>
__global__ void __launch_bounds__(kGnnThreads, 1) gnn_kernel(GnnArgs a) {
  extern __shared__ __align__(16) float sm[];
  constexpr int PF = phase_floats<D>();
  const int p = blockIdx.x;
  const int64_t base = a.node_off[p];
  const int n = (int)(a.node_off[p + 1] - base);
  float* lat = a.lat + (int64_t)p * a.ld_lat;
  if (a.err && a.err[p]) {
    for (int k = threadIdx.x; k < a.gn; k += blockDim.x) lat[k] = __int_as_float(0x7fc00000);
    return;
  }
  float* wbuf = sm;                                  // PF floats (>= gather chunk)
  float* red = wbuf + (PF > 2 * D * 32 + 64 ? PF : 2 * D * 32 + 64);   // [warps][32]
  float* hA; float* hB;
  if (a.smem_state) {
    hA = red + (kGnnThreads / 32) * 32;
    hB = hA + (int64_t)n * D;
  } else {
    hA = a.state + base * D;
    hB = a.state + (a.node_off[gridDim.x] + base) * D;
  }

  // ---- embedding: h0 = tanh(X.We + be) ----
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const float* x = a.feats + (base + i) * a.F;
    float acc[D];
    #pragma unroll
    for (int k = 0; k < D; ++k) acc[k] = a.be[k];
    for (int f = 0; f < a.F; ++f) {
      const float xv = x[f];
      #pragma unroll
      for (int k = 0; k < D; ++k) acc[k] = fmaf(xv, __ldg(a.we + f * D + k), acc[k]);
    }
    #pragma unroll
    for (int k = 0; k < D; k += 4)
      *(float4*)(hA + (int64_t)i * D + k) =
          make_float4(fs_tanh(acc[k]), fs_tanh(acc[k + 1]), fs_tanh(acc[k + 2]), fs_tanh(acc[k + 3]));
  }

  // ---- GRU steps: covalent phase, then non-covalent phase ----
  for (int ph = 0; ph < 2; ++ph) {
    __syncthreads();
    for (int t = threadIdx.x; t < PF; t += blockDim.x) wbuf[t] = a.phase[ph][t];
    __syncthreads();
    const float* Wc = wbuf;
    const float* bc = Wc + D * 3 * D;
    const float* U = bc + 3 * D;
    const float* Uh = U + D * 2 * D;
    const int64_t* rows = ph == 0 ? a.row_cov : a.row_ncov;
    const int32_t* degs = ph == 0 ? a.deg_cov : a.deg_ncov;
    const col_t* cols = ph == 0 ? a.col_cov : a.col_ncov;
    for (int step = 0; step < a.k_steps[ph]; ++step) {
      for (int i = threadIdx.x; i < n; i += blockDim.x) {
        // keep ptxas from hoisting the (loop-invariant) shared-memory weight
        // loads out of the node loop: that would need thousands of registers
        asm volatile("" ::: "memory");
        float h[D], s[D];
        #pragma unroll
        for (int k = 0; k < D; k += 4) {
          float4 v = *(const float4*)(hA + (int64_t)i * D + k);
          h[k] = v.x; h[k + 1] = v.y; h[k + 2] = v.z; h[k + 3] = v.w;
          s[k] = 0.f; s[k + 1] = 0.f; s[k + 2] = 0.f; s[k + 3] = 0.f;
        }
        const int64_t rb = rows[base + i], re = rb + degs[base + i];
        for (int64_t q = rb; q < re; ++q) {
          const float* hj = hA + (int64_t)cols[q] * D;
          #pragma unroll
          for (int k = 0; k < D; k += 4) {
            float4 v = *(const float4*)(hj + k);
            s[k] += v.x; s[k + 1] += v.y; s[k + 2] += v.z; s[k + 3] += v.w;
          }
        }
        // z gate
        float z[D], rh[D];
        #pragma unroll
        for (int k = 0; k < D; ++k) z[k] = bc[k];
        #pragma unroll
        for (int c = 0; c < D; ++c) {
          #pragma unroll
          for (int k = 0; k < D; ++k) z[k] = fmaf(s[c], Wc[c * 3 * D + k], fmaf(h[c], U[c * 2 * D + k], z[k]));
        }
        #pragma unroll
        for (int k = 0; k < D; ++k) rh[k] = bc[D + k];
        #pragma unroll
        for (int c = 0; c < D; ++c) {
          #pragma unroll
          for (int k = 0; k < D; ++k)
            rh[k] = fmaf(s[c], Wc[c * 3 * D + D + k], fmaf(h[c], U[c * 2 * D + D + k], rh[k]));
        }
        #pragma unroll
        for (int k = 0; k < D; ++k) { z[k] = fs_sigmoid(z[k]); rh[k] = fs_sigmoid(rh[k]) * h[k]; }
        float hh[D];
        #pragma unroll
        for (int k = 0; k < D; ++k) hh[k] = bc[2 * D + k];
        #pragma unroll
        for (int c = 0; c < D; ++c) {
          #pragma unroll
          for (int k = 0; k < D; ++k)
            hh[k] = fmaf(s[c], Wc[c * 3 * D + 2 * D + k], fmaf(rh[c], Uh[c * D + k], hh[k]));
        }
        #pragma unroll
        for (int k = 0; k < D; k += 4) {
          float4 o;
          o.x = fmaf(z[k], fs_tanh(hh[k]) - h[k], h[k]);
          o.y = fmaf(z[k + 1], fs_tanh(hh[k + 1]) - h[k + 1], h[k + 1]);
          o.z = fmaf(z[k + 2], fs_tanh(hh[k + 2]) - h[k + 2], h[k + 2]);
          o.w = fmaf(z[k + 3], fs_tanh(hh[k + 3]) - h[k + 3], h[k + 3]);
          *(float4*)(hB + (int64_t)i * D + k) = o;
        }
      }
      __syncthreads();
      float* t = hA; hA = hB; hB = t;
    }
  }

  // ---- gated gather + mean over all nodes of the pose (8 columns / pass) ----
  constexpr int CW = 8;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const float inv_n = 1.0f / (float)max(n, 1);
  for (int c0 = 0; c0 < a.gn; c0 += CW) {
    const int nc = min(CW, a.gn - c0);
    __syncthreads();
    float* Gg = wbuf;            // [D][CW]
    float* Gf = wbuf + D * CW;   // [D][CW]
    float* b2 = wbuf + 2 * D * CW;
    for (int t = threadIdx.x; t < D * CW; t += blockDim.x) {
      const int c = t / CW, k = t % CW;
      Gg[t] = k < nc ? a.gg[c * a.gn + c0 + k] : 0.f;
      Gf[t] = k < nc ? a.gf[c * a.gn + c0 + k] : 0.f;
    }
    for (int t = threadIdx.x; t < CW; t += blockDim.x) {
      b2[t] = t < nc ? a.bg[c0 + t] : 0.f;
      b2[CW + t] = t < nc ? a.bf[c0 + t] : 0.f;
    }
    __syncthreads();
    float acc[CW];
    #pragma unroll
    for (int k = 0; k < CW; ++k) acc[k] = 0.f;
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
      asm volatile("" ::: "memory");
      float gz[CW], fz[CW];
      #pragma unroll
      for (int k = 0; k < CW; ++k) { gz[k] = b2[k]; fz[k] = b2[CW + k]; }
      #pragma unroll
      for (int c = 0; c < D; c += 4) {
        const float4 hv = *(const float4*)(hA + (int64_t)i * D + c);
        const float hc[4] = {hv.x, hv.y, hv.z, hv.w};
        #pragma unroll
        for (int q = 0; q < 4; ++q) {
          #pragma unroll
          for (int k = 0; k < CW; ++k) {
            gz[k] = fmaf(hc[q], Gg[(c + q) * CW + k], gz[k]);
            fz[k] = fmaf(hc[q], Gf[(c + q) * CW + k], fz[k]);
          }
        }
      }
      #pragma unroll
      for (int k = 0; k < CW; ++k) acc[k] = fmaf(fs_sigmoid(gz[k]), fs_tanh(fz[k]), acc[k]);
    }
    // fixed-order reduction: lanes (xor tree) then warps (sequential)
    #pragma unroll
    for (int k = 0; k < CW; ++k) {
      float v = acc[k];
      #pragma unroll
      for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
      acc[k] = v;
    }
    if (lane == 0) {
      #pragma unroll
      for (int k = 0; k < CW; ++k) red[warp * CW + k] = acc[k];
    }
    __syncthreads();
    if (threadIdx.x < nc) {
      float t = 0.f;
      for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += red[w * CW + threadIdx.x];
      lat[c0 + threadIdx.x] = t * inv_n;
    }
  }
}

template <int D>
static size_t gnn_smem_bytes(int max_nodes, bool smem_state) {
  size_t w = phase_floats<D>() > 2 * D * 32 + 64 ? phase_floats<D>() : 2 * D * 32 + 64;
  size_t b = (w + (kGnnThreads / 32) * 32) * 4;
  if (smem_state) b += (size_t)2 * max_nodes * D * 4;
  return b;
}

template <int D>
static int launch_gnn_d(const GnnArgs& a0, int n_poses, int max_nodes, cudaStream_t st) {
  GnnArgs a = a0;
  const size_t limit = 227 * 1024;
  a.smem_state = gnn_smem_bytes<D>(max_nodes, true) <= limit ? 1 : 0;
  if (!a.smem_state && a.state == nullptr) return FS_ECAPACITY;
  const size_t smem = gnn_smem_bytes<D>(max_nodes, a.smem_state);
  FS_CUDA_CHECK(cudaFuncSetAttribute(gnn_kernel<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  gnn_kernel<D><<<n_poses, kGnnThreads, smem, st>>>(a);
  FS_LAUNCH_CHECK();
  return FS_OK;
}

// Padded width the kernels are instantiated for (weights are zero-padded to
// it on the host; zero-padded channels stay exactly zero through every step).
int gnn_padded_width(int d) {
  if (d <= 8) return 8;
  if (d <= 16) return 16;
  if (d <= 24) return 24;
  if (d <= 32) return 32;
  return -1;   // wider node states are not instantiated (reference default: 24)
}

int launch_gnn(const GnnArgs& a, int dpad, int n_poses, int max_nodes, cudaStream_t st) {
  if (n_poses <= 0) return FS_OK;
  switch (dpad) {
    case 8: return launch_gnn_d<8>(a, n_poses, max_nodes, st);
    case 16: return launch_gnn_d<16>(a, n_poses, max_nodes, st);
    case 24: return launch_gnn_d<24>(a, n_poses, max_nodes, st);
    case 32: return launch_gnn_d<32>(a, n_poses, max_nodes, st);
    default: return FS_ENOTSUP;
  }
}

bool gnn_needs_global_state(int dpad, int max_nodes) {
  const size_t limit = 227 * 1024;
  switch (dpad) {
    case 8: return gnn_smem_bytes<8>(max_nodes, true) > limit;
    case 16: return gnn_smem_bytes<16>(max_nodes, true) > limit;
    case 24: return gnn_smem_bytes<24>(max_nodes, true) > limit;
    default: return gnn_smem_bytes<32>(max_nodes, true) > limit;
  }
}

}  // namespace fs
