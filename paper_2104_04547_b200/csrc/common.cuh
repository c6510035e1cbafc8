// Shared device helpers for the fusionb200 kernels (sm_100a).
#pragma once
#include <cstdio>

#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <stdint.h>

#include "../../include/fusionb200.h"

namespace fs {

// Record the last CUDA error per host thread (reported by fs_last_cuda_error),
// with the library source site that saw it.
void set_cuda_error(cudaError_t e, const char* file = nullptr, int line = 0);

#define FS_CUDA_CHECK(expr)                                   \
  do {                                                        \
    cudaError_t _e = (expr);                                  \
    if (_e != cudaSuccess) { ::fs::set_cuda_error(_e, __FILE__, __LINE__); return FS_ECUDA; } \
  } while (0)

// Pose-local neighbour ids of the scoring-path CSR (FS_MAX_POSE_ATOMS < 2^16):
// 16-bit halves the id traffic of the SG-CNN gathers.
typedef uint16_t col_t;

// Device-side index checks, compiled in only with -DFS_BOUNDS (FS_BOUNDS=1 build).
#ifdef FS_BOUNDS
#define FS_DCHECK(cond, what, v, lim)                                                                \
  do {                                                                                             \
    if (!(cond)) {                                                                                 \
      printf("FS_DCHECK %s:%d %s: %lld vs %lld (block %d)\n", __FILE__, __LINE__, what, (long long)(v), \
             (long long)(lim), (int)blockIdx.x);                                                   \
      __trap();                                                                                    \
    }                                                                                              \
  } while (0)
#else
#define FS_DCHECK(cond, what, v, lim) do {} while (0)
#endif

// Kernel launches issued by the library (reported by fs_launch_count()).
// With FS_DEBUG_SYNC=1 in the environment every launch is followed by a
// device synchronise and a report of the launching site on failure.
void count_launch(const char* file, int line);
#define FS_LAUNCH_CHECK()            \
  do {                               \
    ::fs::count_launch(__FILE__, __LINE__); \
    FS_CUDA_CHECK(cudaGetLastError()); \
  } while (0)

// Optional per-stage CUDA events recorded on the launching stream
// (fs_set_stage_events); stage ids below.
enum Stage { ST_FEATURIZE = 0, ST_CONV1, ST_CONV2, ST_CONV3, ST_CONV4, ST_DENSE, ST_GNN, ST_FUSION, ST_END,
             ST_COUNT };
void mark_stage(int stage, cudaStream_t st);

inline int cuda_status(cudaError_t e) {
  if (e != cudaSuccess) { set_cuda_error(e); return FS_ECUDA; }
  return FS_OK;
}

__host__ __device__ inline int64_t cdiv(int64_t a, int64_t b) { return (a + b - 1) / b; }

// ---- pose batch access ---------------------------------------------------
// Pose p's nodes: pocket atoms of pose_target[p] (if any) followed by its own
// atoms; mirrors np.vstack([prot, lig]) (complexes.py:114-118).
struct PoseView {
  const double* pxyz; const int32_t* pelem; const int32_t* prole; int64_t np_;
  const double* axyz; const int32_t* aelem; const int32_t* arole; int64_t na;
  __device__ __forceinline__ int64_t n() const { return np_ + na; }
  __device__ __forceinline__ void atom(int64_t i, double& x, double& y, double& z,
                                       int32_t& e, int32_t& r) const {
    const double* q; int64_t j;
    if (i < np_) { q = pxyz + 3 * i; e = pelem[i]; r = prole[i]; }
    else { j = i - np_; q = axyz + 3 * j; e = aelem[j]; r = arole[j]; }
    x = q[0]; y = q[1]; z = q[2];
  }
};

__device__ __forceinline__ PoseView pose_view(const fs_pose_batch& b, int p) {
  PoseView v;
  int t = (b.pose_target != nullptr) ? b.pose_target[p] : -1;
  if (t >= 0) {
    int64_t s = b.pocket_off[t];
    v.pxyz = b.pocket_xyz + 3 * s; v.pelem = b.pocket_elem + s; v.prole = b.pocket_role + s;
    v.np_ = b.pocket_off[t + 1] - s;
  } else {
    v.pxyz = nullptr; v.pelem = nullptr; v.prole = nullptr; v.np_ = 0;
  }
  int64_t a = b.atom_off[p];
  v.axyz = b.atom_xyz + 3 * a; v.aelem = b.atom_elem + a; v.arole = b.atom_role + a;
  v.na = b.atom_off[p + 1] - a;
  return v;
}

// ---- exact float64 arithmetic (no FMA contraction) ------------------------
__device__ __forceinline__ double dist2_exact(double dx, double dy, double dz) {
  // ((dx*dx + dy*dy) + dz*dz): the cKDTree / np.linalg.norm summation order.
  return __dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz));
}

// ---- activations -----------------------------------------------------------
// Accurate-enough fp32 transcendentals: ex2.approx has ~2 ulp relative error,
// so sigmoid/tanh below carry ~1e-7 absolute error (tanh.approx.f32 would
// carry 2^-11 relative and compound over the 9 GRU steps).
__device__ __forceinline__ float fs_rcp(float x) {
  float r;   // MUFU.RCP: <= 1 ulp, no slow-path call (keeps GEMV loops spill-free)
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}
__device__ __forceinline__ float fs_sigmoid(float x) {
  // 0.5*(1+tanh(x/2)) == 1/(1+exp(-x)) (autodiff.py:322-327)
  return fs_rcp(1.0f + __expf(-x));
}
__device__ __forceinline__ float fs_tanh(float x) {
  // branch-free tanh(x) = 1 - 2/(1 + e^{2x}): absolute error ~1e-7 (what the
  // GRU update h + z*(hh - h) and the gated gather consume)
  const float e = __expf(2.0f * fminf(fmaxf(x, -15.0f), 15.0f));
  return 1.0f - 2.0f * fs_rcp(1.0f + e);
}

// Pre-scaled forms for the tensor-core SG-CNN, whose packed weights and biases
// already carry the exponent scale (so the GEMM output is the ex2 argument):
//   fs_sigmoid_pre(u) = sigmoid(x) with u = -log2(e) x
//   fs_tanh_pre(u)    = tanh(x)    with u = 2 log2(e) x
// ex2(+inf) = inf and rcp(inf) = 0 give the right limits without clamps.
__device__ __forceinline__ float fs_ex2(float u) {
  float r;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(u));
  return r;
}
__device__ __forceinline__ float fs_sigmoid_pre(float u) { return fs_rcp(1.0f + fs_ex2(u)); }
__device__ __forceinline__ float fs_tanh_pre(float u) { return fmaf(-2.0f, fs_rcp(1.0f + fs_ex2(u)), 1.0f); }
constexpr double kNegLog2e = -1.4426950408889634074;
constexpr double kTwoLog2e = 2.8853900817779268147;

#define FS_ACT_NONE 0
#define FS_ACT_RELU 1
#define FS_ACT_LEAKY 2
#define FS_ACT_SELU 3
#define FS_ACT_SIGMOID 4
#define FS_ACT_TANH 5

__device__ __forceinline__ float fs_act(int kind, float x) {
  switch (kind) {
    case FS_ACT_RELU: return fmaxf(x, 0.0f);
    case FS_ACT_LEAKY: return x > 0.0f ? x : 0.01f * x;                 // autodiff.py:303-308
    case FS_ACT_SELU:                                                    // autodiff.py:311-319
      return 1.0507009873554805f * (x > 0.0f ? x : 1.6732632423543772f * expm1f(x));
    case FS_ACT_SIGMOID: return fs_sigmoid(x);
    case FS_ACT_TANH: return fs_tanh(x);
    default: return x;
  }
}

}  // namespace fs
