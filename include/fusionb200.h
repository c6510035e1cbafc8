/*
 * fusionb200 -- C-ABI of the B200-native Coherent-Fusion pose-scoring path.
 *
 * Replaces, for the hot path only, the reference package `fusionscreen`
 * (/root/reference/pkg/src/fusionscreen).  Each entry point names the
 * reference interface it stands in for.  The reference is pure Python, so
 * its "FFI" is the Python operator/plugin API; the binding a maintainer adds
 * is the ctypes layer in INTEGRATION.md (our own package binds it the same
 * way in paper_2104_04547_b200/_native.py).
 *
 * Conventions
 *   - C types only; no exceptions cross the ABI; every function returns an
 *     int status (FS_OK == 0, negative on error, see fs_strerror()).
 *   - Every array argument is a CALLER-OWNED DEVICE pointer unless the
 *     parameter name starts with `host_`.  The library never allocates or
 *     frees caller memory; scratch comes from a caller-provided workspace
 *     sized by fs_workspace_bytes().
 *   - Every launch takes a cudaStream_t (passed as void*) and is
 *     stream-ordered and asynchronous.  No call synchronises the device.
 *   - Reentrant: no mutable globals; a packed weight blob is immutable, so
 *     several host threads may score concurrently on separate streams
 *     (SPEC.md:298 -- frozen models are safe for concurrent prediction).
 *   - Per-pose item failures are reported in an int32 err[P] bit mask and
 *     never abort the batch (models.py:470-498 contract).
 */
#ifndef FUSIONB200_H
#define FUSIONB200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes ----------------------------------------------------- */
#define FS_OK         0
#define FS_EINVAL    -1   /* bad argument (ValueError in the reference)   */
#define FS_ECAPACITY -2   /* workspace / per-pose size limit exceeded      */
#define FS_ECUDA     -3   /* CUDA runtime error                            */
#define FS_ENOTSUP   -4   /* configuration not supported by this precision */

/* ---- per-pose error bits (int32 err[P]) -------------------------------- */
#define FS_ERR_ROLE       1  /* role not in {PROTEIN=0, LIGAND=1}           */
#define FS_ERR_NAN        2  /* NaN coordinate (voxelize raises, :180-183)  */
#define FS_ERR_NONFINITE  4  /* +-inf/NaN coordinate -> non-finite features */
#define FS_ERR_EDGE_CAP   8  /* CSR workspace overflow: retry, larger cap   */
#define FS_ERR_TOO_LARGE 16  /* pose exceeds FS_MAX_POSE_ATOMS              */
#define FS_ERR_GRID_NONFINITE 32  /* given voxel grid has inf/NaN (models.py:521-522) */
#define FS_ERR_FEAT_NONFINITE 64  /* given node features have inf/NaN (:527-528)   */
#define FS_ERR_NOT_FACTORED 128   /* fs_score_poses_cached: pose is not pocket(role 0)
                                     + ligand(role 1) or its ligand is too large for
                                     the factored kernels; rescore with fs_score_poses */

#define FS_MAX_POSE_ATOMS 4096

/* ---- precision of the scoring path ------------------------------------ */
/* The precision argument alone fixes every arithmetic choice of a call (no
 * environment knobs change numerics).
 *   FS_PREC_FP32  : FFMA fp32 everywhere (the reference within 1e-3 relative;
 *                   measured ~1e-7).  Slow: the correctness anchor.
 *   FS_PREC_BF16  : the throughput path.  tcgen05 Conv3d on bf16 operands and
 *                   bf16 activations (fp32 TMEM accumulation), tcgen05 kind::tf32
 *                   dense1, SG-CNN GEMMs on mma.sync with fp16 hi/lo activations
 *                   x fp16 weights (2 passes, fp32 accumulate; transcendentals
 *                   via ex2.approx / tanh.approx in the pool), fp32 fusion MLP.
 *                   Stated tolerance vs the reference: see DESIGN.md section 4.
 *   FS_PREC_MIXED : fp32-class on the tensor cores (the 1e-3 path).  Every
 *                   tensor-core GEMM is a 3-pass bf16 split (x = hi + lo,
 *                   A.B ~ Alo.Bhi + Ahi.Blo + Ahi.Bhi, fp32 accumulate): tcgen05
 *                   Conv3d with activations carried as (hi, lo) bf16 pairs and
 *                   hi/lo weight sets, SG-CNN GEMMs on mma.sync likewise with
 *                   fp32 node states and accurate ex2/rcp gates; dense1 FFMA
 *                   fp32; fp32 fusion MLP. */
#define FS_PREC_FP32  0
#define FS_PREC_BF16  1
#define FS_PREC_MIXED 2

/* ---- grid layouts ------------------------------------------------------ */
#define FS_GRID_NCDHW_F64  0  /* reference VoxelGrid.occupancy [C,G,G,G] f64 */
#define FS_GRID_NDHWC_F32  1  /* conv input, fp32, channels innermost        */
#define FS_GRID_NDHWC_BF16 2  /* conv input, bf16, channels innermost        */

/* A batch of poses.  Pose p's nodes are: the pocket atoms of target
 * pose_target[p] (if pose_target != NULL and pose_target[p] >= 0), followed
 * by atoms atom_off[p] .. atom_off[p+1]-1.  This is exactly the reference's
 * `np.vstack([prot, lig])` node order (complexes.py:114-118) when the pocket
 * holds the protein atoms; a plain SyntheticComplex is a pose with no pocket.
 * Coordinates are float64 [n,3] (complexes.py:74); elements and roles int32. */
typedef struct {
  const double*  pocket_xyz;
  const int32_t* pocket_elem;
  const int32_t* pocket_role;
  const int64_t* pocket_off;   /* [n_pockets+1] */
  int32_t        n_pockets;
  const double*  atom_xyz;
  const int32_t* atom_elem;
  const int32_t* atom_role;
  const int64_t* atom_off;     /* [n_poses+1] */
  const int32_t* pose_target;  /* [n_poses] or NULL */
  int32_t        n_poses;
  int32_t        max_pose_atoms; /* upper bound on nodes of any pose (host-known) */
} fs_pose_batch;

/* Model configuration: the union of VoxelHeadConfig (models.py:40-63),
 * GraphHeadConfig (:66-93) and FusionConfig (:96-118) fields that affect
 * inference, plus the featurizer box size (models.py:638-642). */
typedef struct {
  int32_t grid_extent, in_channels, conv_filters_1, conv_filters_2;
  int32_t dense_nodes, kernel_1, kernel_2;
  int32_t residual_1, residual_2, batch_norm;
  int32_t c_elem, k_cov, k_noncov, gather_width_cov, gather_width_noncov;
  double  cov_thresh, noncov_thresh, box_size;
  int32_t fusion_mode;          /* 0 late, 1 mid, 2 coherent               */
  int32_t n_fusion_layers, model_specific_layers, residual_fusion;
  int32_t activation;           /* 0 relu, 1 leaky-relu, 2 selu            */
  int32_t fusion_dense_nodes;
} fs_model_desc;

#define FS_MODE_LATE 0
#define FS_MODE_MID 1
#define FS_MODE_COHERENT 2

/* Packed device weight blob (immutable after fs_pack_weights).  Holds fp32
 * copies in kernel layouts plus bf16 UMMA-layout conv weights. */
typedef struct fs_model fs_model;

/* ---- library ------------------------------------------------------------ */
const char* fs_strerror(int code);
int fs_version(void);
/* Last CUDA error string seen by this thread (diagnostics). */
const char* fs_last_cuda_error(void);
/* Number of kernel launches the library has issued (process-wide). */
long long fs_launch_count(void);
/* Optional per-stage timing for fs_score_poses on the calling thread:
 * `events` is an array of 9 cudaEvent_t (featurize, conv1, conv2, conv3,
 * conv4, dense, gnn, fusion, end) recorded on the scoring stream at each
 * stage boundary; NULL disables.  Entries may be NULL. */
int fs_set_stage_events(void** events, int n);
/* Branch scheduling of fs_score_poses / fs_score_poses_cached on the calling
 * thread: 0 serial on the caller's stream, 1 radius graph on a side stream,
 * 2 voxel branch on a high-priority side stream (the default), -1 = the
 * FS_OVERLAP environment default.  Results are bitwise identical in every
 * mode; serial mode makes the per-stage events exact per-kernel times. */
int fs_set_overlap(int mode);

/* ---- weights (FusionModel.__init__/load -> device) ---------------------- */
/* Replaces FusionModel parameter binding (models.py:263-278, :441-467).
 * host_names/host_params: the reference parameter dict flattened as
 * "voxel/<name>", "graph/<name>", "fusion/<name>" (models.py:532-539), fp64,
 * shapes as in init_*_params (models.py:150-218).  Optional BN running stats
 * "voxel/bn1_mean", "voxel/bn1_var", "voxel/bn2_mean", "voxel/bn2_var".
 * Creates a host handle; device memory is the caller's `dev_blob` of
 * fs_weights_bytes() bytes, filled asynchronously on `stream`. */
size_t fs_weights_bytes(const fs_model_desc* desc);
int fs_model_create(const fs_model_desc* desc, const char* const* host_names,
                    const double* const* host_params, int n_params,
                    void* dev_blob, size_t blob_bytes, void* stream,
                    fs_model** out);
int fs_model_destroy(fs_model* m);
/* 1 if `precision` is implemented for this model's configuration. */
int fs_model_supports(const fs_model* m, int precision);

/* ---- featurizer (complexes.py:171-254) --------------------------------- */
/* node_off[P+1] (int64) of a pose batch; required by the graph calls. */
int fs_node_offsets(const fs_pose_batch* b, int64_t* node_off, void* ws,
                    size_t ws_bytes, void* stream);
size_t fs_node_offsets_ws_bytes(int32_t n_poses);

/* voxelize (complexes.py:171-184) for every pose; `out` layout per
 * FS_GRID_*; err[p] |= FS_ERR_ROLE / FS_ERR_NAN.  Output is overwritten. */
int fs_voxelize(const fs_pose_batch* b, int32_t extent, int32_t c_elem,
                double box_size, int32_t layout, void* out, int32_t* err,
                void* stream);

/* Node features [onehot(clip elem) | role | pos/box+0.5] (complexes.py:233-236),
 * float64 [N, c_elem+4]. */
int fs_node_features(const fs_pose_batch* b, const int64_t* node_off,
                     int32_t c_elem, double box_size, double* out, void* stream);

/* Radius graph (complexes.py:237-246), two passes.
 * count: deg_cov/deg_ncov [N] = per-node degrees of the symmetric adjacency.
 * fill:  CSR rows row_cov/row_ncov [N+1] (int64, global entry offsets) are
 *        produced by fs_graph_rows; col_* hold POSE-LOCAL neighbour ids,
 *        each row sorted ascending; dist_* (nullable) the float64 distances.
 * Predicate (exact, float64, no FMA): d2 = (dx*dx+dy*dy)+dz*dz;
 *   edge iff d2 <= rmax*rmax and sqrt(d2) <= t_role (rmax = max(t_cov,t_ncov)). */
int fs_graph_count(const fs_pose_batch* b, const int64_t* node_off,
                   double cov_thresh, double noncov_thresh,
                   int32_t* deg_cov, int32_t* deg_ncov, int32_t* err,
                   void* stream);
int fs_graph_rows(const int32_t* deg, int64_t n_nodes, int64_t* row_ptr,
                  void* ws, size_t ws_bytes, void* stream);
size_t fs_graph_rows_ws_bytes(int64_t n_nodes);
int fs_graph_fill(const fs_pose_batch* b, const int64_t* node_off,
                  double cov_thresh, double noncov_thresh,
                  const int64_t* row_cov, const int64_t* row_ncov,
                  int32_t* col_cov, int32_t* col_ncov,
                  double* dist_cov, double* dist_ncov,
                  int64_t cap_cov, int64_t cap_ncov, int32_t* err, void* stream);
/* Extract the i<j edge list (lexsorted) of one CSR: edges [E,2] (pose-local
 * node ids, int64) and dists.  `edge_off` [P+1] int64 from fs_graph_edge_counts. */
int fs_graph_edge_counts(const int64_t* node_off, int32_t n_poses,
                         const int64_t* row_ptr, const int32_t* col,
                         int64_t* edge_off, void* ws, size_t ws_bytes,
                         void* stream);
int fs_graph_edges(const int64_t* node_off, int32_t n_poses,
                   const int64_t* row_ptr, const int32_t* col, const double* dist,
                   const int64_t* edge_off, int64_t* edges, double* dists,
                   void* stream);

/* Inspection of the SCORING-PATH radius graph (the edge lists north_star
 * requires bit-exact): runs the graph exactly as the scoring call does --
 * fs_score_poses's node offsets + fused single-launch CSR kernel, or with
 * `factored` != 0 fs_score_poses_cached's pocket-factored kernel (ligand-ligand
 * covalent + ligand-pocket non-covalent edges; pocket-pocket edges live in the
 * pocket cache) -- then lists every DIRECTED CSR entry the SG-CNN would read:
 * ent_*[(p * max_edges + k) * 2 + {0,1}] = (i, j), k < n_*[p], pose-local
 * node ids in the pose's original numbering (pocket atoms, then its own),
 * with the float64 distance sqrt((dx*dx+dy*dy)+dz*dz) in d_* (nullable).
 * Replaces nothing in the reference; it exposes what build_graph
 * (complexes.py:237-246) computes on the scoring path for parity tests.
 * Workspace: fs_scoring_graph_ws_bytes(P, max_pose_atoms, max_edges,
 * factored, c_elem).  err[P] as fs_score_poses (FS_ERR_NOT_FACTORED when a
 * pose cannot be factored). */
size_t fs_scoring_graph_ws_bytes(int32_t n_poses, int32_t max_pose_atoms, int64_t max_edges, int32_t factored,
                                 int32_t c_elem);
int fs_scoring_graph(const fs_pose_batch* b, double cov_thresh, double noncov_thresh, int64_t max_edges,
                     int32_t factored, int32_t max_pocket_atoms, int32_t c_elem, double box_size, void* ws,
                     size_t ws_bytes, int32_t* n_cov, int32_t* n_ncov, int32_t* ent_cov, int32_t* ent_ncov,
                     double* d_cov, double* d_ncov, int32_t* err, void* stream);

/* ---- scoring (FusionModel.predict_batch, models.py:470-498) ------------ */
/* Workspace for fs_score_poses / fs_score_poses_cached: max_nodes =
 * max_poses * (per-pose node bound: the batch's max_pose_atoms, or the
 * factored slice rows), max_edges = max_poses * the per-pose edge cap. */
size_t fs_workspace_bytes(const fs_model* m, int32_t max_poses,
                          int64_t max_nodes, int64_t max_edges, int precision);
/* Workspace for fs_score_features: the batch's total nodes and the larger of
 * its two i<j edge counts. */
size_t fs_features_workspace_bytes(const fs_model* m, int32_t n_poses, int64_t n_nodes, int32_t max_pose_nodes,
                                   int64_t n_edges, int precision);

/* Fused featurize + 3D-CNN + SG-CNN + fusion for raw poses (the screening
 * path: models.featurize (:638-651) then predict_batch).  Outputs (nullable
 * except scores) are float32 device arrays: scores[P], lat_v[P,latent_v],
 * lat_g[P,latent_g], pred_v[P], pred_g[P].  err[P] bit mask; poses with
 * err != 0 get NaN score.  max_edges bounds the directed CSR entries of ONE
 * pose per edge type (size the workspace with P*max_edges); a pose above it
 * gets FS_ERR_EDGE_CAP (host retries with a larger bound). */
int fs_score_poses(const fs_model* m, int precision, const fs_pose_batch* b,
                   int64_t max_edges, void* ws, size_t ws_bytes,
                   float* scores, float* lat_v, float* lat_g, float* pred_v,
                   float* pred_g, int32_t* err, void* stream);

/* Pre-featurized batch: the drop-in predict_batch / voxel_head_forward /
 * graph_head_forward path.  grids: float64 [P,C,G,G,G] (VoxelGrid layout,
 * nullable when only the graph head is wanted); feats: float64
 * [N, c_elem+4]; node_off [P+1]; max_pose_nodes = the largest pose's node
 * count (sizes the SG-CNN's on-chip node state; poses above it get
 * FS_ERR_TOO_LARGE; <= 0: unknown, worst case assumed); edges given as i<j pairs with GLOBAL node
 * ids (int64 [E,2]) per edge type.  heads: bit0 voxel head, bit1 graph head,
 * bit2 fusion. */
int fs_score_features(const fs_model* m, int precision, int32_t n_poses,
                      const double* grids, const double* feats,
                      const int64_t* node_off, int64_t n_nodes, int32_t max_pose_nodes,
                      const int64_t* cov_edges, int64_t n_cov,
                      const int64_t* ncov_edges, int64_t n_ncov, int32_t heads,
                      void* ws, size_t ws_bytes, float* scores, float* lat_v,
                      float* lat_g, float* pred_v, float* pred_g, int32_t* err,
                      void* stream);

/* ---- pocket-invariant factoring (one-pocket screens) ---
 * For a pose = pocket atoms (all role PROTEIN) + ligand atoms (all LIGAND) the
 * following never depend on the ligand: the protein voxel channels and their
 * conv1 contribution (conv1 is linear, channels are disjoint,
 * complexes.py:182); protein-protein covalent edges and the protein node
 * states after the covalent phase (covalent edges never cross roles,
 * complexes.py:242-243); and the whole trajectory (and pool contribution) of
 * protein nodes with no ligand within noncov_thresh.  fs_pocket_prepare
 * computes these once per pocket into a cache; fs_score_poses_cached then
 * scores a pose from its ligand atoms, recomputing only ligand nodes and the
 * protein nodes the ligand touches.  Same scores as fs_score_poses to fp32
 * rounding (FS_PREC_BF16 / FS_PREC_MIXED).  This is an effective-throughput mode: the
 * reported algorithmic work per pose is unchanged. */
size_t fs_pocket_cache_bytes(const fs_model* m, int32_t max_pocket_atoms);
size_t fs_pocket_prepare_ws_bytes(const fs_model* m, int32_t n_pockets, int32_t max_pocket_atoms);
/* precision: FS_PREC_BF16 or FS_PREC_MIXED; a cache is used only with the
 * precision it was prepared with (the cached pocket node states come from
 * that precision's SG-CNN).
 * Pockets as in fs_pose_batch (pocket_xyz/elem/role, pocket_off[n+1]); cache =
 * n_pockets * fs_pocket_cache_bytes(max_pocket_atoms) bytes; err[n_pockets]
 * gets the FS_ERR_* bits of each pocket (a pocket with err != 0 must not be
 * used with the cache). */
int fs_pocket_prepare(const fs_model* m, int precision, const double* pocket_xyz, const int32_t* pocket_elem,
                      const int32_t* pocket_role, const int64_t* pocket_off, int32_t n_pockets,
                      int32_t max_pocket_atoms, void* cache, int32_t* err, void* ws,
                      size_t ws_bytes, void* stream);
/* Like fs_score_poses (FS_PREC_BF16 / FS_PREC_MIXED) for a batch whose pockets are the ones the
 * cache was prepared from.  Poses that cannot be factored get
 * FS_ERR_NOT_FACTORED (and a NaN score); rescore them with fs_score_poses.
 * Workspace: fs_workspace_bytes(m, P, P * (max_pose_atoms + 32), P * max_edges, bf16). */
int fs_score_poses_cached(const fs_model* m, int precision, const fs_pose_batch* b,
                          const void* cache, int32_t max_pocket_atoms, int64_t max_edges,
                          void* ws, size_t ws_bytes, float* scores, float* lat_v,
                          float* lat_g, float* pred_v, float* pred_g, int32_t* err,
                          void* stream);

/* Test hook: one tcgen05 Conv3d layer (1..4) of the bf16 voxel head on
 * explicit buffers.  bf16 activations are chunk-major [P][C/8][D][H][W][8]
 * (layer 1 input = the NDHWC bf16 voxel grid, C = 8).  Outputs: 1 -> bf16
 * [P,4,16,16,16,8]; 2 -> bf16 max-pooled [P,4,8,8,8,8]; 3 -> bf16
 * [P,8,8,8,8,8]; 4 -> f32 pooled NDHWC [P,4,4,4,64] with `residual` = layer-3
 * output (h3) added after ReLU. */
int fs_debug_conv(const fs_model* m, int layer, int32_t n_poses, const void* in,
                  const void* residual, void* out, void* stream);

/* ---- ranking (top-k merge; tie rule of evaluate.py:67-83) -------------- */
/* Sorts the concatenation of (a) and (b) by (score desc, index asc) and keeps
 * the first k into (out_scores, out_idx).  NaN scores rank last.  Indices
 * are full int64 (screens past 2^32 poses keep the lowest-index tie rule).
 * Either input may be empty. */
size_t fs_topk_ws_bytes(int64_t n);
int fs_topk_merge(const float* a_scores, const int64_t* a_idx, int64_t na,
                  const float* b_scores, const int64_t* b_idx, int64_t nb,
                  int32_t k, float* out_scores, int64_t* out_idx, void* ws,
                  size_t ws_bytes, void* stream);

/* Per-compound best pose (evaluate.aggregate_best_pose, :67-83) on device:
 * compound[n] int64 ids in [0, n_compounds) (runs need not be contiguous),
 * pose_id[n] (< 2^32); direction +1 max / -1 min.  best_idx[n_compounds] =
 * winning row (-1 if the compound has no rows); best_key[n_compounds] is
 * caller scratch. */
int fs_best_pose(const int64_t* compound, const int64_t* pose_id,
                 const float* scores, int64_t n, int64_t n_compounds,
                 int32_t direction, int64_t* best_idx, uint64_t* best_key,
                 void* stream);

/* Streaming best pose for screens: fold a batch of (compound, pose_id, score)
 * rows into best_key[n_compounds] (row compound c -> slot c - compound_base;
 * rows outside the range are ignored).  best_key must start all-ones
 * (0xff bytes).  Same rule as evaluate.aggregate_best_pose (:67-83).  Then
 * decode to (best_score, best_pose) per compound (-1 / NaN: no rows). */
int fs_best_pose_update(const int64_t* compound, int64_t compound_base,
                        const int64_t* pose_id, const float* scores, int64_t n,
                        int64_t n_compounds, int32_t direction, uint64_t* best_key,
                        void* stream);
int fs_best_pose_decode(const uint64_t* best_key, int64_t n_compounds,
                        int32_t direction, float* best_score, int64_t* best_pose,
                        void* stream);

#ifdef __cplusplus
}
#endif
#endif /* FUSIONB200_H */
