// tcgen05 (UMMA) implicit-GEMM Conv3d chain for the default voxel head
// (bf16 operands, fp32 accumulation in TMEM).  See umma_conv.cu.
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stddef.h>

#include "../../include/fusionb200.h"

namespace fs {
namespace umma {

// True if the voxel-head configuration matches the specialised kernels
// (G=16, Cin=8, filters 32/64, kernels 5/3, residual_2 only, no BN).
bool supports(const fs_model_desc& d);
size_t weights_bytes(const fs_model_desc& d);
// Pack reference fp64 conv weights [O][C][k][k][k] into the UMMA blob.
void pack_weights(const fs_model_desc& d, const double* c1, const double* c2, const double* c3,
                  const double* c4, char* out);
size_t workspace_bytes(const fs_model_desc& d, int64_t n_poses, bool x3 = false);
// grid: [P][G][G][G][Cin] bf16 -> pooled conv4 output [P][(G/4)^3][f2] fp32
// (NDHWC flatten order, ready for dense1).
int voxel_convs(const fs_model_desc& d, const char* wblob, const float* b1, const float* b2,
                const float* b3, const float* b4, int n_poses, const __nv_bfloat16* grid, char* ws,
                float* flat_out, cudaStream_t st);

// The same chain for FS_PREC_MIXED: fp32-class 3-pass hi/lo split on the
// tcgen05 tensor cores (activations as hi/lo bf16 pairs; see umma_conv.cu).
// Workspace: workspace_bytes(d, P, true).
int voxel_convs_x3(const fs_model_desc& d, const char* wblob, const float* b1, const float* b2,
                   const float* b3, const float* b4, int n_poses, const __nv_bfloat16* grid,
                   const __nv_bfloat16* grid_lo, char* ws, float* flat_out, cudaStream_t st);

// The act1 buffer inside the voxel_convs workspace, and conv2..4 from it
// (pocket-factored path: act1 comes from conv1_fact_kernel).
__nv_bfloat16* act1_ptr(char* ws);
int voxel_convs_from2(const fs_model_desc& d, const char* wblob, const float* b2, const float* b3,
                      const float* b4, int n_poses, char* ws, float* flat_out, cudaStream_t st);

// X3 forms (FS_PREC_MIXED): the lo half of act1 in the x3 workspace, and
// conv2..4 from an act1 (hi, lo) pair produced elsewhere.
__nv_bfloat16* act1_lo_ptr(char* ws, int64_t n_poses);
int voxel_convs_from2_x3(const fs_model_desc& d, const char* wblob, const float* b2, const float* b3,
                         const float* b4, int n_poses, char* ws, float* flat_out, cudaStream_t st);

// One layer (1..4) on explicit buffers, for per-layer parity tests.
int debug_layer(const fs_model_desc& d, const char* wblob, const float* bias, const float* unused, int layer, int P,
                const void* in, const void* residual, void* out, cudaStream_t st);

// dense1 on tcgen05 kind::tf32: y[P][N] = relu(x[P][K] . W + b) with
// wt = W^T [N][K]; x must hold dense_rows_padded(P) rows.  N == 128 only.
bool dense_tf32_ok(int K, int N);
size_t dense_rows_padded(int64_t P);
int dense_tf32(const float* x, int P, int K, const float* wt, int N, const float* bias, float* y, cudaStream_t st);

}  // namespace umma
}  // namespace fs
