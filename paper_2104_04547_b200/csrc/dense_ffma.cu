// FP32 (FFMA) kernels of the reference-accurate path: generic Conv3d, 2^3
// max-pool and a strided dense/GEMM with fused epilogue.
//
// Reference ops: conv3d (autodiff.py:208-232), max-pool3d (:251-269),
// dense (:161-173) + relu/leaky/selu (:298-319), elementwise-add (:447-456).
// Layout: activations are NDHWC float32 ([P][D][H][W][C]); conv weights are
// packed [kd][kh][kw][C][O] (cross-correlation, zero "same" padding).
#include "common.cuh"

namespace fs {

// ---------------------------------------------------------------------------
// Conv3d, FFMA.  Block = 32 voxels (lanes) x ceil(O/8) warps; each thread
// owns 8 output channels of one voxel.  Weight reads are warp-uniform
// (broadcast); input reads are reused across the O/8 warps through L1.
// Epilogue: relu(acc + b) [* bn_scale + bn_shift] [+ residual].
// ---------------------------------------------------------------------------
struct ConvArgs {
  const float* in; const float* w; const float* b;
  const float* bn_scale; const float* bn_shift; const float* residual;
  float* out;
  int64_t n_vox;      // P * G^3
  int g, cin, cout, k;
  int no_relu;        // 1: out = acc + b (pocket cache: conv1 pre-activation)
};

__global__ void __launch_bounds__(256) conv3d_ffma_kernel(ConvArgs a) {
  const int lane = threadIdx.x & 31, og = threadIdx.x >> 5;
  const int64_t v = (int64_t)blockIdx.x * 32 + lane;
  const int o0 = og * 8;
  if (v >= a.n_vox || o0 >= a.cout) return;
  const int g = a.g, r = a.k / 2;
  const int64_t g3 = (int64_t)g * g * g;
  const int64_t p = v / g3;
  const int rem = (int)(v - p * g3);
  const int d = rem / (g * g), h = (rem / g) % g, w = rem % g;
  float acc[8];
  #pragma unroll
  for (int q = 0; q < 8; ++q) acc[q] = 0.0f;
  const float* inp = a.in + p * g3 * a.cin;
  const int nvalid = min(8, a.cout - o0);
  for (int i = 0; i < a.k; ++i) {
    const int dd = d + i - r;
    if (dd < 0 || dd >= g) continue;
    for (int j = 0; j < a.k; ++j) {
      const int hh = h + j - r;
      if (hh < 0 || hh >= g) continue;
      for (int l = 0; l < a.k; ++l) {
        const int ww = w + l - r;
        if (ww < 0 || ww >= g) continue;
        const float* x = inp + (((int64_t)dd * g + hh) * g + ww) * a.cin;
        const float* wk = a.w + (((int64_t)(i * a.k + j) * a.k + l) * a.cin) * a.cout + o0;
        if (nvalid == 8 && (a.cout & 3) == 0) {
          for (int c = 0; c < a.cin; ++c) {
            const float xv = __ldg(x + c);
            const float4 w0 = __ldg((const float4*)(wk + (int64_t)c * a.cout));
            const float4 w1 = __ldg((const float4*)(wk + (int64_t)c * a.cout + 4));
            acc[0] = fmaf(xv, w0.x, acc[0]); acc[1] = fmaf(xv, w0.y, acc[1]);
            acc[2] = fmaf(xv, w0.z, acc[2]); acc[3] = fmaf(xv, w0.w, acc[3]);
            acc[4] = fmaf(xv, w1.x, acc[4]); acc[5] = fmaf(xv, w1.y, acc[5]);
            acc[6] = fmaf(xv, w1.z, acc[6]); acc[7] = fmaf(xv, w1.w, acc[7]);
          }
        } else {
          for (int c = 0; c < a.cin; ++c) {
            const float xv = __ldg(x + c);
            #pragma unroll
            for (int q = 0; q < 8; ++q)
              if (q < nvalid) acc[q] = fmaf(xv, __ldg(wk + (int64_t)c * a.cout + q), acc[q]);
          }
        }
      }
    }
  }
  float* o = a.out + v * a.cout + o0;
  #pragma unroll
  for (int q = 0; q < 8; ++q) {
    if (q >= nvalid) break;
    float y = a.no_relu ? acc[q] + a.b[o0 + q] : fmaxf(acc[q] + a.b[o0 + q], 0.0f);
    if (a.bn_scale) y = fmaf(y, a.bn_scale[o0 + q], a.bn_shift[o0 + q]);
    if (a.residual) y += a.residual[v * a.cout + o0 + q];
    o[q] = y;
  }
}

int launch_conv3d_ffma(const ConvArgs& a, cudaStream_t st) {
  if (a.n_vox <= 0) return FS_OK;
  const int warps = (a.cout + 7) / 8;
  if (warps > 8) return FS_ENOTSUP;   // cout <= 64 (reference defaults: 32 / 64)
  conv3d_ffma_kernel<<<(unsigned)cdiv(a.n_vox, 32), warps * 32, 0, st>>>(a);
  FS_LAUNCH_CHECK();
  return FS_OK;
}

// ---------------------------------------------------------------------------
// non-overlapping 2^3 max-pool, NDHWC (autodiff.py:251-269)
// ---------------------------------------------------------------------------
__global__ void maxpool2_kernel(const float* in, float* out, int64_t n_out, int g_out, int c) {
  int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n_out) return;
  const int ch = (int)(t % c);
  int64_t vo = t / c;
  const int64_t go3 = (int64_t)g_out * g_out * g_out;
  const int64_t p = vo / go3;
  const int rem = (int)(vo - p * go3);
  const int d = rem / (g_out * g_out), h = (rem / g_out) % g_out, w = rem % g_out;
  const int gi = 2 * g_out;
  const float* base = in + p * (int64_t)gi * gi * gi * c;
  float m = -INFINITY;
  #pragma unroll
  for (int i = 0; i < 2; ++i)
    #pragma unroll
    for (int j = 0; j < 2; ++j)
      #pragma unroll
      for (int l = 0; l < 2; ++l)
        m = fmaxf(m, base[(((int64_t)(2 * d + i) * gi + 2 * h + j) * gi + 2 * w + l) * c + ch]);
  out[t] = m;
}

int launch_maxpool2(const float* in, float* out, int n_poses, int g_out, int c, cudaStream_t st) {
  const int64_t n = (int64_t)n_poses * g_out * g_out * g_out * c;
  if (n <= 0) return FS_OK;
  maxpool2_kernel<<<(unsigned)cdiv(n, 256), 256, 0, st>>>(in, out, n, g_out, c);
  FS_LAUNCH_CHECK();
  return FS_OK;
}

// ---------------------------------------------------------------------------
// Dense: Y[m, y_off + n] = act(X[m, :K] . W[K, N] + b[n]) (+ R[m, n]).
// 64x64 output tile per 256-thread block, 4x4 per thread, K tiles of 16.
// ---------------------------------------------------------------------------
struct DenseArgs {
  const float* x; int64_t ldx;
  const float* w; const float* b;   // W [K][N] row-major (reference [in, out])
  const float* r; int64_t ldr;      // residual (nullable)
  float* y; int64_t ldy;
  int64_t m; int k, n; int act;
};

__global__ void __launch_bounds__(256) dense_kernel(DenseArgs a) {
  __shared__ float xs[16][64 + 4];
  __shared__ float ws[16][64 + 4];
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  const int64_t m0 = (int64_t)blockIdx.y * 64;
  const int n0 = blockIdx.x * 64;
  float acc[4][4];
  #pragma unroll
  for (int i = 0; i < 4; ++i)
    #pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = 0.0f;
  for (int k0 = 0; k0 < a.k; k0 += 16) {
    for (int t = threadIdx.x; t < 16 * 64; t += 256) {
      const int kk = t & 15, mm = t >> 4;
      const int64_t gm = m0 + mm;
      const int gk = k0 + kk;
      xs[kk][mm] = (gm < a.m && gk < a.k) ? a.x[gm * a.ldx + gk] : 0.0f;
      const int nn = t & 63, kr = t >> 6;
      const int gn = n0 + nn, gk2 = k0 + kr;
      ws[kr][nn] = (gn < a.n && gk2 < a.k) ? a.w[(int64_t)gk2 * a.n + gn] : 0.0f;
    }
    __syncthreads();
    #pragma unroll
    for (int kk = 0; kk < 16; ++kk) {
      float xv[4], wv[4];
      #pragma unroll
      for (int i = 0; i < 4; ++i) xv[i] = xs[kk][ty * 4 + i];
      #pragma unroll
      for (int j = 0; j < 4; ++j) wv[j] = ws[kk][tx * 4 + j];
      #pragma unroll
      for (int i = 0; i < 4; ++i)
        #pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(xv[i], wv[j], acc[i][j]);
    }
    __syncthreads();
  }
  #pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int64_t gm = m0 + ty * 4 + i;
    if (gm >= a.m) continue;
    #pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int gn = n0 + tx * 4 + j;
      if (gn >= a.n) continue;
      float v = fs_act(a.act, acc[i][j] + (a.b ? a.b[gn] : 0.0f));
      if (a.r) v += a.r[gm * a.ldr + gn];
      a.y[gm * a.ldy + gn] = v;
    }
  }
}

int launch_dense(const DenseArgs& a, cudaStream_t st) {
  if (a.m <= 0 || a.n <= 0) return FS_OK;
  dim3 grid((unsigned)cdiv(a.n, 64), (unsigned)cdiv(a.m, 64));
  dense_kernel<<<grid, 256, 0, st>>>(a);
  FS_LAUNCH_CHECK();
  return FS_OK;
}

// late fusion (models.py:399-405) and invalid-pose masking
__global__ void finalize_kernel(int n, int mode, const float* pv, const float* pg, float* scores,
                                const int32_t* err) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  if (mode == FS_MODE_LATE) scores[i] = (pv[i] + pg[i]) * 0.5f;
  if (err && err[i]) scores[i] = __int_as_float(0x7fc00000);
}

int launch_finalize(int n, int mode, const float* pv, const float* pg, float* scores,
                    const int32_t* err, cudaStream_t st) {
  if (n <= 0) return FS_OK;
  finalize_kernel<<<(int)cdiv(n, 256), 256, 0, st>>>(n, mode, pv, pg, scores, err);
  FS_LAUNCH_CHECK();
  return FS_OK;
}

// f64 VoxelGrid [P,C,G,G,G] -> f32 / bf16 NDHWC conv input
__global__ void grid_f64_to_ndhwc_kernel(const double* in, void* out, int64_t n, int c, int g3,
                                         int bf16, int32_t* err) {
  int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n) return;
  const int ch = (int)(t % c);
  const int64_t vo = t / c;
  const int64_t p = vo / g3;
  const int s = (int)(vo - p * g3);
  double v = in[(p * c + ch) * g3 + s];
  if (err && !isfinite(v)) atomicOr(&err[p], FS_ERR_GRID_NONFINITE);
  if (bf16) ((__nv_bfloat16*)out)[t] = __float2bfloat16_rn((float)v);
  else ((float*)out)[t] = (float)v;
}

int launch_grid_convert(const double* in, void* out, int n_poses, int c, int g, bool bf16,
                        int32_t* err, cudaStream_t st) {
  const int g3 = g * g * g;
  const int64_t n = (int64_t)n_poses * c * g3;
  if (n <= 0) return FS_OK;
  grid_f64_to_ndhwc_kernel<<<(unsigned)cdiv(n, 256), 256, 0, st>>>(in, out, n, c, g3, bf16 ? 1 : 0, err);
  FS_LAUNCH_CHECK();
  return FS_OK;
}

__global__ void f64_to_f32_kernel(const double* in, float* out, int64_t n, int row, const int32_t* node_pose,
                                  int32_t* err) {
  int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n) return;
  double v = in[t];
  if (err && !isfinite(v)) atomicOr(&err[node_pose[t / row]], FS_ERR_FEAT_NONFINITE);
  out[t] = (float)v;
}

// poses above the caller's per-pose node bound are flagged (the SG-CNN sizes
// its shared-memory node state by that bound and skips flagged poses)
__global__ void pose_bound_kernel(const int64_t* node_off, int n_poses, int64_t bound, int32_t* err) {
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p < n_poses && node_off[p + 1] - node_off[p] > bound) atomicOr(&err[p], FS_ERR_TOO_LARGE);
}

int launch_pose_bound(const int64_t* node_off, int n_poses, int64_t bound, int32_t* err, cudaStream_t st) {
  if (n_poses <= 0) return FS_OK;
  pose_bound_kernel<<<(unsigned)cdiv(n_poses, 256), 256, 0, st>>>(node_off, n_poses, bound, err);
  FS_LAUNCH_CHECK();
  return FS_OK;
}

// fp32 -> (hi, lo) bf16 pair: hi = bf16(x), lo = bf16(x - hi) (the X3 operands)
__global__ void split_bf16_kernel(const float* in, __nv_bfloat16* hi, __nv_bfloat16* lo, int64_t n) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n) return;
  const float x = in[t];
  const __nv_bfloat16 h = __float2bfloat16_rn(x);
  hi[t] = h;
  lo[t] = __float2bfloat16_rn(x - __bfloat162float(h));
}

int launch_split_bf16(const float* in, __nv_bfloat16* hi, __nv_bfloat16* lo, int64_t n, cudaStream_t st) {
  if (n <= 0) return FS_OK;
  split_bf16_kernel<<<(unsigned)cdiv(n, 256), 256, 0, st>>>(in, hi, lo, n);
  FS_LAUNCH_CHECK();
  return FS_OK;
}

int launch_f64_to_f32(const double* in, float* out, int64_t n, int row, const int32_t* node_pose,
                      int32_t* err, cudaStream_t st) {
  if (n <= 0) return FS_OK;
  f64_to_f32_kernel<<<(unsigned)cdiv(n, 256), 256, 0, st>>>(in, out, n, row, node_pose, err);
  FS_LAUNCH_CHECK();
  return FS_OK;
}

}  // namespace fs
