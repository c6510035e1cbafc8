// tcgen05 implicit-GEMM Conv3d (placeholder until the UMMA kernels land).
#include "common.cuh"
#include "umma_conv.cuh"

namespace fs {
namespace umma {

bool supports(const fs_model_desc&) { return false; }
size_t weights_bytes(const fs_model_desc&) { return 0; }
void pack_weights(const fs_model_desc&, const double*, const double*, const double*, const double*, char*) {}
size_t workspace_bytes(const fs_model_desc&, int64_t) { return 0; }
int voxel_convs(const fs_model_desc&, const char*, const float*, const float*, const float*, const float*, int,
                const __nv_bfloat16*, char*, float*, cudaStream_t) {
  return FS_ENOTSUP;
}

}  // namespace umma
}  // namespace fs
