// SG-CNN on the tensor cores (gnn_mma.cu): launch arguments shared with abi.cu.
#pragma once
#include "common.cuh"

namespace fs {

struct GnnMmaArgs {
  const float* feats; int F;
  const int64_t* node_off;
  const int64_t* row_cov; const int32_t* deg_cov; const col_t* col_cov;     // row start + degree
  const int64_t* row_ncov; const int32_t* deg_ncov; const col_t* col_ncov;
  const float* we; const float* be;       // [F][24], [24]
  const uint32_t* wfrag[2];               // per phase, see gnn_mma_phase_words()
  const float* wbias[2];                  // per phase [72] = bz | br | bh
  const uint32_t* gfrag;                  // gather fragments [2 hi/lo][2 kt][32 nt][32][2]
  const uint32_t* wfrag16[2];             // fp16 phase fragments (SPLIT 2), [zr | hh] in the hi layout
  const uint32_t* gfrag16;                // fp16 gather fragments (SPLIT 2)
  const float* gbias;                     // [256] = bg | bf (ex2-scaled, SPLIT 3)
  const float* wbias16[2];                // SPLIT 2 phase biases [72], tanh-scaled like wfrag16
  const float* gbias16;                   // SPLIT 2 pool biases [256], tanh-scaled like gfrag16
  int k_steps[2];
  float* lat; int64_t ld_lat;             // [P][ld_lat], columns 0..127
  const int32_t* err;
  // ---- pocket factoring (fs_score_poses_cached); fact_cnt == nullptr: off.
  // Pose p owns node slice [p*fact_stride, +fact_stride): ligand rows
  // [0, nL), zero rows up to nLp = roundup16(nL), then the nA pocket atoms
  // the ligand touches (ids fact_aff[]), whose covalent phase is taken from
  // the pocket cache (cache_hcov) and whose untouched neighbours enter the
  // pool through cache_T - sum(cache_f[affected]).
  const int32_t* fact_cnt;                // [P][2] = (nL, nA)
  int64_t fact_stride;
  const int32_t* fact_aff;                // [P*fact_stride]
  const int32_t* pose_target;             // [P]
  const char* cache; int64_t cache_stride;
  int64_t off_hcov, off_f, off_T, off_n;  // byte offsets inside one pocket's cache
  // ---- pocket preparation dumps (plain path): node states after the covalent
  // phase [P][dump_ld][24] and per-node pool terms [P][dump_ld][128]
  float* dump_hcov; float* dump_f; int64_t dump_ld;
  int heavy_cap;                          // rows of the heavy-sum buffer (set by launch_gnn_mma)
  int ids_padded;                         // CSR rows padded to 4 ids with the zero row (graph_csr.cu)
};

int gnn_mma_phase_words();
int gnn_mma_gather_words();
bool gnn_mma_fits(int max_nodes);
int gnn_mma_max_nodes();
int launch_gnn_mma(const GnnMmaArgs& a, int split, int n_poses, int max_nodes, cudaStream_t st);

}  // namespace fs
