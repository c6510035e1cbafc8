// C-ABI of libfusionb200: weight packing, workspace planning and the scoring
// pipelines (featurize -> 3D-CNN -> SG-CNN -> fusion) on one CUDA stream.
//
// Reference call stack being replaced: FusionModel.predict_batch
// (models.py:470-498) -> build_tape (:441-467) -> _voxel_tape (:285-322),
// _graph_tape (:351-371), _fusion_tape (:374-396); featurize (:638-651) ->
// voxelize / build_graph (complexes.py:171-254).
#include <atomic>
#include <cmath>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <map>
#include <string>
#include <vector>

#include <cuda_fp16.h>

#include "common.cuh"
#include "gnn_mma.cuh"
#include "umma_conv.cuh"

namespace fs {

static thread_local std::string g_last_cuda_error;
void set_cuda_error(cudaError_t e, const char* file, int line) {
  g_last_cuda_error = cudaGetErrorString(e);
  if (file) {
    const char* base = strrchr(file, '/');
    g_last_cuda_error += std::string(" at ") + (base ? base + 1 : file) + ":" + std::to_string(line);
  }
}

static std::atomic<long long> g_launches{0};
void count_launch(const char* file, int line) {
  g_launches.fetch_add(1, std::memory_order_relaxed);
  static const bool dbg = getenv("FS_DEBUG_SYNC") != nullptr;
  if (dbg) {
    const cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) fprintf(stderr, "fusionb200: launch at %s:%d failed: %s\n", file, line, cudaGetErrorString(e));
  }
}

static thread_local cudaEvent_t* g_stage_events = nullptr;   // [ST_COUNT] or null
void mark_stage(int stage, cudaStream_t st) {
  if (!g_stage_events || !g_stage_events[stage]) return;
  // inside a CUDA-graph capture the record must be an external (timed) node
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  cudaStreamIsCapturing(st, &cs);
  if (cs == cudaStreamCaptureStatusActive)
    cudaEventRecordWithFlags(g_stage_events[stage], st, cudaEventRecordExternal);
  else
    cudaEventRecord(g_stage_events[stage], st);
}

// ---- launchers defined in the other translation units ----------------------
int launch_node_offsets(const fs_pose_batch& b, int64_t* node_off, void* ws, size_t ws_bytes, cudaStream_t st,
                        int64_t clamp = 0);
int launch_voxelize(const fs_pose_batch& b, int g, int c_elem, double box, int layout, void* out, int32_t* err, cudaStream_t st);
int launch_node_features(const fs_pose_batch& b, const int64_t* node_off, int c_elem, double box, void* out, bool f64, cudaStream_t st);
int launch_graph_count(const fs_pose_batch& b, const int64_t* node_off, double tc, double tn, int32_t* deg_cov, int32_t* deg_ncov, int32_t* err, cudaStream_t st);
int launch_graph_fill(const fs_pose_batch& b, const int64_t* node_off, double tc, double tn, const int64_t* row_cov, const int64_t* row_ncov, int32_t* col_cov, int32_t* col_ncov, double* dist_cov, double* dist_ncov, int64_t cap_cov, int64_t cap_ncov, int32_t* err, cudaStream_t st);
int launch_rows(const int32_t* deg, int64_t n, int64_t* row_ptr, void* ws, size_t ws_bytes, cudaStream_t st);
int launch_edge_counts(const int64_t* node_off, int n_poses, const int64_t* row_ptr, const int32_t* col, int64_t* edge_off, void* ws, size_t ws_bytes, cudaStream_t st);
int launch_edges(const int64_t* node_off, int n_poses, const int64_t* row_ptr, const int32_t* col, const double* dist, const int64_t* edge_off, int64_t* edges, double* dists, cudaStream_t st);
int launch_graph_csr(const fs_pose_batch& b, const int64_t* node_off, double tc, double tn, int64_t* row_cov,
                     int32_t* deg_cov, col_t* col_cov, double* dist_cov, int64_t* row_ncov, int32_t* deg_ncov,
                     col_t* col_ncov, double* dist_ncov, int64_t cap, int32_t* err, cudaStream_t st,
                     float* feats = nullptr, int c_elem = 0, double box = 0.0);
int launch_graph_fact(const fs_pose_batch& b, double tc, double tn, double box, int c_elem, int64_t S, int64_t cap,
                      int max_pocket, int32_t* cnt, int32_t* aff, float* feats, int64_t* row_cov, int32_t* deg_cov,
                      col_t* col_cov, int64_t* row_ncov, int32_t* deg_ncov, col_t* col_ncov, int32_t* err,
                      cudaStream_t st);
int launch_csr_entries(const fs_pose_batch& b, const int64_t* node_off, const int32_t* fact_cnt, const int32_t* aff,
                       int64_t S, int64_t cap, int max_rows, const int64_t* row_cov, const int32_t* deg_cov,
                       const col_t* col_cov, const int64_t* row_ncov, const int32_t* deg_ncov, const col_t* col_ncov,
                       int64_t cap_out, int32_t* n_cov, int32_t* n_ncov, int32_t* ent_cov, int32_t* ent_ncov,
                       double* d_cov, double* d_ncov, const int32_t* err, cudaStream_t st);
bool conv1_fact_supported(int g, int k, int cin, int cout);
int launch_conv1_fact(const fs_pose_batch& b, const char* cache, int64_t cache_stride, int64_t off_pp,
                      int64_t off_ppact, int64_t off_wl, int c_elem, double box, __nv_bfloat16* out, cudaStream_t st,
                      int64_t off_ppact_lo, __nv_bfloat16* out_lo);
int launch_pocket_conv1_fields(const float* pp, int n_pockets, char* cache, int64_t cache_stride, int64_t off_ppact,
                               int64_t off_wl, const float* w1, int c_elem, cudaStream_t st, int64_t off_ppact_lo,
                               int x3);
int launch_round_bf16(const float* in, float* out, int64_t n, cudaStream_t st);
int launch_pocket_total(const int64_t* pocket_off, int n_pockets, const float* f, int64_t ld, char* cache,
                        int64_t cache_stride, int64_t off_T, int64_t off_n, cudaStream_t st);
int launch_pocket_poses(int n, int64_t* atom_off, int32_t* target, cudaStream_t st);
int launch_csr_from_edges(const int64_t* edges, int64_t ne, const int64_t* node_off, int n_poses, int64_t n_nodes, int32_t* node_pose, int32_t* deg, int64_t* row_ptr, int64_t* cursor, col_t* col, void* ws, size_t ws_bytes, cudaStream_t st);
size_t scan_ws_bytes(int64_t n);

struct ConvArgs {
  const float* in; const float* w; const float* b;
  const float* bn_scale; const float* bn_shift; const float* residual;
  float* out; int64_t n_vox; int g, cin, cout, k; int no_relu;
};
int launch_conv3d_ffma(const ConvArgs& a, cudaStream_t st);
int launch_maxpool2(const float* in, float* out, int n_poses, int g_out, int c, cudaStream_t st);
struct DenseArgs {
  const float* x; int64_t ldx; const float* w; const float* b;
  const float* r; int64_t ldr; float* y; int64_t ldy; int64_t m; int k, n; int act;
};
int launch_dense(const DenseArgs& a, cudaStream_t st);
int launch_finalize(int n, int mode, const float* pv, const float* pg, float* scores, const int32_t* err, cudaStream_t st);
int launch_grid_convert(const double* in, void* out, int n_poses, int c, int g, bool bf16, int32_t* err, cudaStream_t st);
int launch_f64_to_f32(const double* in, float* out, int64_t n, int row, const int32_t* node_pose, int32_t* err, cudaStream_t st);
int launch_split_bf16(const float* in, __nv_bfloat16* hi, __nv_bfloat16* lo, int64_t n, cudaStream_t st);
int launch_pose_bound(const int64_t* node_off, int n_poses, int64_t bound, int32_t* err, cudaStream_t st);

struct GnnArgs {
  const float* feats; int F; const int64_t* node_off;
  const int64_t* row_cov; const int32_t* deg_cov; const col_t* col_cov;
  const int64_t* row_ncov; const int32_t* deg_ncov; const col_t* col_ncov;
  const float* we; const float* be; const float* phase[2];
  const float* gg; const float* bg; const float* gf; const float* bf;
  int k_steps[2]; int gn; float* state; float* lat; int64_t ld_lat; const int32_t* err; int smem_state;
};
int gnn_padded_width(int d);
int launch_gnn(const GnnArgs& a, int dpad, int n_poses, int max_nodes, cudaStream_t st);
bool gnn_needs_global_state(int dpad, int max_nodes);

size_t topk_ws_bytes(int64_t n);
int launch_topk_merge(const float* as, const int64_t* ai, int64_t na, const float* bs, const int64_t* bi, int64_t nb, int k, float* os, int64_t* oi, void* ws, size_t ws_bytes, cudaStream_t st);
int launch_best_pose(const int64_t* compound, const int64_t* pose_id, const float* s, int64_t n, int64_t n_compounds, int dir, int64_t* best_idx, uint64_t* best_key, cudaStream_t st);
int launch_best_update(const int64_t* compound, int64_t base, const int64_t* pose_id, const float* s, int64_t n, int64_t n_compounds, int dir, uint64_t* best_key, cudaStream_t st);
int launch_best_decode(const uint64_t* best_key, int64_t n, int dir, float* score, int64_t* pose, cudaStream_t st);

static inline size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

// ---------------------------------------------------------------------------
// weight blob layout (float offsets; every block 64-float aligned)
// ---------------------------------------------------------------------------
struct Layout {
  size_t n = 0;
  size_t take(size_t floats) { size_t o = n; n = align_up(n + floats, 64); return o; }
};

}  // namespace fs

struct fs_model {
  fs_model_desc d;
  float* blob = nullptr;
  size_t blob_bytes = 0;
  int cin, f1, f2, k1, k2, G, dn, lv, flat, gn, dg, dpad, F, w1, w2, fd, LW, cgrid;
  size_t c1w, c1b, c2w, c2b, c3w, c3b, c4w, c4b, bn1s, bn1h, bn2s, bn2h;
  size_t d1w, d1b, d1t, d2w, d2b, ow, ob;   // d1t: dense1 W^T [dn][flat] (tcgen05 dense1)
  size_t we, be, ph[2], gg, bg, gf, bf, gd1w, gd1b, gd2w, gd2b, gow, gob;
  size_t msg, msgb, msv, msvb, fw[8], fb[8];
  size_t umma_off = 0;   // byte offset of the bf16 UMMA conv weights
  bool umma_ok = false;
  bool gmma_ok = false;  // tensor-core SG-CNN (widths 24 / 128)
  size_t gm_wf[2], gm_wb[2], gm_gf, gm_gb;
  size_t gm_wf16[2], gm_gf16;   // fp16 weight fragments of the 2-pass SG-CNN
  size_t gm_wb16[2], gm_gb16;   // its biases (tanh-scaled like the fp16 fragments)
  const float* P(size_t off) const { return blob + off; }
};

namespace fs {

static int validate_desc(const fs_model_desc& d) {
  if (d.grid_extent < 8 || d.grid_extent % 4) return FS_EINVAL;
  if (d.in_channels < 1 || d.conv_filters_1 < 1 || d.conv_filters_2 < 1) return FS_EINVAL;
  if (d.conv_filters_1 > 64 || d.conv_filters_2 > 64) return FS_ENOTSUP;
  if (d.kernel_1 < 1 || d.kernel_2 < 1 || !(d.kernel_1 & 1) || !(d.kernel_2 & 1)) return FS_EINVAL;
  if (d.dense_nodes < 2) return FS_EINVAL;
  if (d.c_elem < 1 || d.c_elem + 4 > 64) return FS_EINVAL;
  if (d.k_cov < 2 || d.k_cov > 8 || d.k_noncov < 2 || d.k_noncov > 8) return FS_EINVAL;  // models.py:76-79
  if (gnn_padded_width(d.gather_width_cov) < 0 || d.gather_width_cov < 1) return FS_ENOTSUP;
  if (d.gather_width_noncov < 2) return FS_EINVAL;
  if (d.fusion_mode < 0 || d.fusion_mode > 2) return FS_EINVAL;
  if (d.fusion_mode != FS_MODE_LATE && (d.n_fusion_layers < 3 || d.n_fusion_layers > 5)) return FS_EINVAL;
  if (d.activation < 0 || d.activation > 2) return FS_EINVAL;
  if (!(d.cov_thresh >= 1.2 && d.cov_thresh <= 5.9) || !(d.noncov_thresh >= 1.2 && d.noncov_thresh <= 5.9))
    return FS_EINVAL;
  return FS_OK;
}

static size_t plan_model(fs_model& m) {
  const fs_model_desc& d = m.d;
  m.cin = d.in_channels; m.f1 = d.conv_filters_1; m.f2 = d.conv_filters_2;
  m.k1 = d.kernel_1; m.k2 = d.kernel_2; m.G = d.grid_extent; m.dn = d.dense_nodes;
  m.lv = d.dense_nodes / 2; m.flat = m.f2 * (m.G / 4) * (m.G / 4) * (m.G / 4);
  m.gn = d.gather_width_noncov; m.dg = d.gather_width_cov; m.dpad = gnn_padded_width(m.dg);
  m.F = d.c_elem + 4; m.w1 = (int)(m.gn / 1.5); m.w2 = m.w1 / 2;
  m.fd = d.fusion_dense_nodes; m.cgrid = d.in_channels / 2;
  m.LW = d.model_specific_layers && d.fusion_mode != FS_MODE_LATE ? 2 * (m.gn + m.lv) : (m.gn + m.lv);
  Layout L;
  m.c1w = L.take((size_t)m.k1 * m.k1 * m.k1 * m.cin * m.f1); m.c1b = L.take(m.f1);
  m.c2w = L.take((size_t)m.k2 * m.k2 * m.k2 * m.f1 * m.f1); m.c2b = L.take(m.f1);
  m.c3w = L.take((size_t)m.k2 * m.k2 * m.k2 * m.f1 * m.f2); m.c3b = L.take(m.f2);
  m.c4w = L.take((size_t)m.k2 * m.k2 * m.k2 * m.f2 * m.f2); m.c4b = L.take(m.f2);
  m.bn1s = L.take(m.f1); m.bn1h = L.take(m.f1); m.bn2s = L.take(m.f2); m.bn2h = L.take(m.f2);
  m.d1w = L.take((size_t)m.flat * m.dn); m.d1b = L.take(m.dn); m.d1t = L.take((size_t)m.flat * m.dn);
  m.d2w = L.take((size_t)m.dn * m.lv); m.d2b = L.take(m.lv);
  m.ow = L.take(m.lv); m.ob = L.take(1);
  const int D = m.dpad;
  m.we = L.take((size_t)m.F * D); m.be = L.take(D);
  for (int ph = 0; ph < 2; ++ph) m.ph[ph] = L.take((size_t)6 * D * D + 3 * D);
  m.gg = L.take((size_t)D * m.gn); m.bg = L.take(m.gn);
  m.gf = L.take((size_t)D * m.gn); m.bf = L.take(m.gn);
  m.gd1w = L.take((size_t)m.gn * m.w1); m.gd1b = L.take(m.w1);
  m.gd2w = L.take((size_t)m.w1 * m.w2); m.gd2b = L.take(m.w2);
  m.gow = L.take(m.w2); m.gob = L.take(1);
  if (d.fusion_mode != FS_MODE_LATE) {
    if (d.model_specific_layers) {
      m.msg = L.take((size_t)m.gn * m.gn); m.msgb = L.take(m.gn);
      m.msv = L.take((size_t)m.lv * m.lv); m.msvb = L.take(m.lv);
    }
    int width = m.LW;
    for (int i = 0; i < d.n_fusion_layers; ++i) {
      int out = i + 1 < d.n_fusion_layers ? m.fd : 1;
      m.fw[i] = L.take((size_t)width * out); m.fb[i] = L.take(out);
      width = out;
    }
  }
  m.gmma_ok = m.dg == 24 && m.gn == 128;
  if (m.gmma_ok) {
    for (int ph = 0; ph < 2; ++ph) { m.gm_wf[ph] = L.take(gnn_mma_phase_words()); m.gm_wb[ph] = L.take(72); }
    m.gm_gf = L.take(gnn_mma_gather_words());
    m.gm_gb = L.take(256);
    for (int ph = 0; ph < 2; ++ph) m.gm_wf16[ph] = L.take(gnn_mma_phase_words() / 2);
    m.gm_gf16 = L.take(gnn_mma_gather_words() / 2);
    for (int ph = 0; ph < 2; ++ph) m.gm_wb16[ph] = L.take(72);
    m.gm_gb16 = L.take(256);
  }
  size_t bytes = L.n * 4;
  m.umma_ok = umma::supports(d);
  if (m.umma_ok) {
    m.umma_off = align_up(bytes, 1024);
    bytes = m.umma_off + umma::weights_bytes(d);
  }
  return align_up(bytes, 256);
}

struct ParamMap {
  std::map<std::string, const double*> p;
  const double* get(const char* name) const {
    auto it = p.find(name);
    return it == p.end() ? nullptr : it->second;
  }
};

static int pack_model(fs_model& m, const ParamMap& pm, std::vector<float>& h) {
  const fs_model_desc& d = m.d;
  h.assign(m.blob_bytes / 4, 0.0f);
  auto need = [&](const char* n) -> const double* { return pm.get(n); };
  // conv [O][C][k][k][k] -> [kd][kh][kw][C][O]
  auto pack_conv = [&](const char* wn, const char* bn, size_t wo, size_t bo, int O, int C, int k) -> int {
    const double* w = need(wn); const double* b = need(bn);
    if (!w || !b) return FS_EINVAL;
    for (int o = 0; o < O; ++o)
      for (int c = 0; c < C; ++c)
        for (int i = 0; i < k; ++i)
          for (int j = 0; j < k; ++j)
            for (int l = 0; l < k; ++l)
              h[wo + ((((size_t)i * k + j) * k + l) * C + c) * O + o] =
                  (float)w[((((size_t)o * C + c) * k + i) * k + j) * k + l];
    for (int o = 0; o < O; ++o) h[bo + o] = (float)b[o];
    return FS_OK;
  };
  int rc;
  if ((rc = pack_conv("voxel/conv1_w", "voxel/conv1_b", m.c1w, m.c1b, m.f1, m.cin, m.k1))) return rc;
  if ((rc = pack_conv("voxel/conv2_w", "voxel/conv2_b", m.c2w, m.c2b, m.f1, m.f1, m.k2))) return rc;
  if ((rc = pack_conv("voxel/conv3_w", "voxel/conv3_b", m.c3w, m.c3b, m.f2, m.f1, m.k2))) return rc;
  if ((rc = pack_conv("voxel/conv4_w", "voxel/conv4_b", m.c4w, m.c4b, m.f2, m.f2, m.k2))) return rc;
  if (d.batch_norm) {
    // eval batch norm folded to y*scale + shift (autodiff.py:335-368; eps 1e-5)
    const char* names[2][4] = {{"voxel/bn1_gamma", "voxel/bn1_beta", "voxel/bn1_mean", "voxel/bn1_var"},
                               {"voxel/bn2_gamma", "voxel/bn2_beta", "voxel/bn2_mean", "voxel/bn2_var"}};
    size_t so[2] = {m.bn1s, m.bn2s}, ho[2] = {m.bn1h, m.bn2h};
    int cs[2] = {m.f1, m.f2};
    for (int q = 0; q < 2; ++q) {
      const double* g = need(names[q][0]); const double* be = need(names[q][1]);
      const double* mu = need(names[q][2]); const double* var = need(names[q][3]);
      if (!g || !be) return FS_EINVAL;
      for (int c = 0; c < cs[q]; ++c) {
        double mean = mu ? mu[c] : 0.0, v = var ? var[c] : 1.0;
        double sc = g[c] / std::sqrt(v + 1e-5);
        h[so[q] + c] = (float)sc;
        h[ho[q] + c] = (float)(be[c] - mean * sc);
      }
    }
  }
  // dense1 rows: reference flatten order (c, d, h, w) (autodiff.py:549-553) ->
  // NDHWC order (d, h, w, c)
  {
    const double* w = need("voxel/dense1_w"); const double* b = need("voxel/dense1_b");
    if (!w || !b) return FS_EINVAL;
    const int S = m.G / 4, C = m.f2;
    for (int c = 0; c < C; ++c)
      for (int s = 0; s < S * S * S; ++s) {
        size_t ref = (size_t)c * S * S * S + s, ours = (size_t)s * C + c;
        for (int n = 0; n < m.dn; ++n) h[m.d1w + ours * m.dn + n] = (float)w[ref * m.dn + n];
      }
    for (int n = 0; n < m.dn; ++n) h[m.d1b + n] = (float)b[n];
    for (int n = 0; n < m.dn; ++n)
      for (int k = 0; k < m.flat; ++k) h[m.d1t + (size_t)n * m.flat + k] = h[m.d1w + (size_t)k * m.dn + n];
  }
  auto copy = [&](const char* n, size_t off, size_t count) -> int {
    const double* w = need(n);
    if (!w) return FS_EINVAL;
    for (size_t i = 0; i < count; ++i) h[off + i] = (float)w[i];
    return FS_OK;
  };
  if ((rc = copy("voxel/dense2_w", m.d2w, (size_t)m.dn * m.lv))) return rc;
  if ((rc = copy("voxel/dense2_b", m.d2b, m.lv))) return rc;
  if ((rc = copy("voxel/out_w", m.ow, m.lv))) return rc;
  if ((rc = copy("voxel/out_b", m.ob, 1))) return rc;
  // graph head, zero-padded to D = dpad
  {
    const int D = m.dpad, dg = m.dg;
    const double* ew = need("graph/embed_w"); const double* eb = need("graph/embed_b");
    if (!ew || !eb) return FS_EINVAL;
    for (int f = 0; f < m.F; ++f)
      for (int k = 0; k < dg; ++k) h[m.we + (size_t)f * D + k] = (float)ew[(size_t)f * dg + k];
    for (int k = 0; k < dg; ++k) h[m.be + k] = (float)eb[k];
    const char* phases[2] = {"cov", "noncov"};
    for (int ph = 0; ph < 2; ++ph) {
      char nm[64];
      auto g = [&](const char* s) { snprintf(nm, sizeof nm, "graph/%s_%s", phases[ph], s); return need(nm); };
      const double* msg = g("msg_w");
      const double* W[3] = {g("wz"), g("wr"), g("wh")};
      const double* U[3] = {g("uz"), g("ur"), g("uh")};
      const double* B[3] = {g("bz"), g("br"), g("bh")};
      if (!msg) return FS_EINVAL;
      for (int q = 0; q < 3; ++q) if (!W[q] || !U[q] || !B[q]) return FS_EINVAL;
      float* base = &h[m.ph[ph]];
      float* Wc = base; float* bc = Wc + 3 * D * D; float* Uc = bc + 3 * D; float* Uh = Uc + 2 * D * D;
      for (int q = 0; q < 3; ++q)
        for (int c = 0; c < dg; ++c)
          for (int k = 0; k < dg; ++k) {
            double acc = 0.0;   // W_msg . W_gate folded in float64
            for (int t = 0; t < dg; ++t) acc += msg[(size_t)c * dg + t] * W[q][(size_t)t * dg + k];
            Wc[(size_t)c * 3 * D + q * D + k] = (float)acc;
          }
      for (int q = 0; q < 3; ++q)
        for (int k = 0; k < dg; ++k) bc[q * D + k] = (float)B[q][k];
      for (int c = 0; c < dg; ++c)
        for (int k = 0; k < dg; ++k) {
          Uc[(size_t)c * 2 * D + k] = (float)U[0][(size_t)c * dg + k];
          Uc[(size_t)c * 2 * D + D + k] = (float)U[1][(size_t)c * dg + k];
          Uh[(size_t)c * D + k] = (float)U[2][(size_t)c * dg + k];
        }
    }
    const double* ggw = need("graph/gather_gate_w"); const double* ggb = need("graph/gather_gate_b");
    const double* gfw = need("graph/gather_feat_w"); const double* gfb = need("graph/gather_feat_b");
    if (!ggw || !ggb || !gfw || !gfb) return FS_EINVAL;
    for (int c = 0; c < dg; ++c)
      for (int k = 0; k < m.gn; ++k) {
        h[m.gg + (size_t)c * m.gn + k] = (float)ggw[(size_t)c * m.gn + k];
        h[m.gf + (size_t)c * m.gn + k] = (float)gfw[(size_t)c * m.gn + k];
      }
    for (int k = 0; k < m.gn; ++k) { h[m.bg + k] = (float)ggb[k]; h[m.bf + k] = (float)gfb[k]; }
  }
  if (m.gmma_ok) {
    // m16n8k16 B fragments (bf16 hi/lo): word0 = (W[16kt+2t][8nt+g], W[16kt+2t+1][8nt+g]),
    // word1 = (W[16kt+2t+8][8nt+g], W[16kt+2t+9][8nt+g]); lane = 4g + t.
    auto bf16_bits = [](double x) -> uint32_t {
      float f = (float)x;
      uint32_t u;
      std::memcpy(&u, &f, 4);
      if ((u & 0x7f800000u) != 0x7f800000u) u += 0x7fffu + ((u >> 16) & 1u);
      return u >> 16;
    };
    auto bf16_val = [&](double x) -> double {
      uint32_t b = bf16_bits(x) << 16;
      float f;
      std::memcpy(&f, &b, 4);
      return (double)f;
    };
    auto frags = [&](const std::vector<double>& W, int K, int N, uint32_t* out_hi, uint32_t* out_lo) {
      const int KT = K / 16, NT = N / 8;
      for (int kt = 0; kt < KT; ++kt)
        for (int nt = 0; nt < NT; ++nt)
          for (int lane = 0; lane < 32; ++lane) {
            const int g = lane >> 2, t = lane & 3;
            const int n = 8 * nt + g;
            const int ks[4] = {16 * kt + 2 * t, 16 * kt + 2 * t + 1, 16 * kt + 2 * t + 8, 16 * kt + 2 * t + 9};
            uint32_t hi[4], lo[4];
            for (int e = 0; e < 4; ++e) {
              const double w = W[(size_t)ks[e] * N + n];
              hi[e] = bf16_bits(w);
              lo[e] = bf16_bits(w - bf16_val(w));
            }
            const size_t o = ((size_t)(kt * NT + nt) * 32 + lane) * 2;
            out_hi[o] = hi[0] | (hi[1] << 16);
            out_hi[o + 1] = hi[2] | (hi[3] << 16);
            out_lo[o] = lo[0] | (lo[1] << 16);
            out_lo[o + 1] = lo[2] | (lo[3] << 16);
          }
    };
    // fp16 fragments in the layout of the bf16 "hi" set (2-pass SG-CNN)
    auto frags16 = [&](const std::vector<double>& W, int K, int N, uint32_t* out) {
      const int KT = K / 16, NT = N / 8;
      for (int kt = 0; kt < KT; ++kt)
        for (int nt = 0; nt < NT; ++nt)
          for (int lane = 0; lane < 32; ++lane) {
            const int g = lane >> 2, t = lane & 3;
            const int n = 8 * nt + g;
            const int ks[4] = {16 * kt + 2 * t, 16 * kt + 2 * t + 1, 16 * kt + 2 * t + 8, 16 * kt + 2 * t + 9};
            uint32_t hv[4];
            for (int e = 0; e < 4; ++e) {
              const __half hb = __float2half_rn((float)W[(size_t)ks[e] * N + n]);
              uint16_t u;
              std::memcpy(&u, &hb, 2);
              hv[e] = u;
            }
            const size_t o = ((size_t)(kt * NT + nt) * 32 + lane) * 2;
            out[o] = hv[0] | (hv[1] << 16);
            out[o + 1] = hv[2] | (hv[3] << 16);
          }
    };
    const char* phases[2] = {"cov", "noncov"};
    const int dg = 24;
    for (int ph = 0; ph < 2; ++ph) {
      char nm[64];
      auto g = [&](const char* s) { snprintf(nm, sizeof nm, "graph/%s_%s", phases[ph], s); return need(nm); };
      const double* msg = g("msg_w");
      const double* W[3] = {g("wz"), g("wr"), g("wh")};
      const double* U[3] = {g("uz"), g("ur"), g("uh")};
      const double* B[3] = {g("bz"), g("br"), g("bh")};
      auto fold = [&](int q, int c, int k) {
        double acc = 0.0;
        for (int t2 = 0; t2 < dg; ++t2) acc += msg[(size_t)c * dg + t2] * W[q][(size_t)t2 * dg + k];
        return acc;
      };
      // gate pre-activations carry the scale of their activation:
      //  bf16 sets (3-pass): the ex2 scale (fs_sigmoid_pre / fs_tanh_pre),
      //   z, r by -log2(e), h~ by 2 log2(e);
      //  fp16 set (2-pass): the tanh scale, z, r by 1/2 (sigmoid(x) =
      //   (1 + tanh(x/2)) / 2), h~ by 1 -- exact power-of-two scalings
      auto pack = [&](const double (&sc)[3], std::vector<double>& Wzr, std::vector<double>& Whh) {
        for (int c = 0; c < 24; ++c)
          for (int k = 0; k < 24; ++k) {
            Wzr[(size_t)c * 48 + k] = sc[0] * fold(0, c, k);
            Wzr[(size_t)c * 48 + 24 + k] = sc[1] * fold(1, c, k);
            Wzr[(size_t)(24 + c) * 48 + k] = sc[0] * U[0][(size_t)c * dg + k];
            Wzr[(size_t)(24 + c) * 48 + 24 + k] = sc[1] * U[1][(size_t)c * dg + k];
            Whh[(size_t)c * 24 + k] = sc[2] * fold(2, c, k);
            Whh[(size_t)(24 + c) * 24 + k] = sc[2] * U[2][(size_t)c * dg + k];
          }
      };
      std::vector<double> Wzr((size_t)48 * 48), Whh((size_t)48 * 24);
      const double sc[3] = {kNegLog2e, kNegLog2e, kTwoLog2e};
      pack(sc, Wzr, Whh);
      uint32_t* wf = reinterpret_cast<uint32_t*>(&h[m.gm_wf[ph]]);
      const int zr = 3 * 6 * 64, hh = 3 * 3 * 64;
      frags(Wzr, 48, 48, wf, wf + zr);
      frags(Whh, 48, 24, wf + 2 * zr, wf + 2 * zr + hh);
      for (int q = 0; q < 3; ++q)
        for (int k = 0; k < 24; ++k) h[m.gm_wb[ph] + q * 24 + k] = (float)(sc[q] * B[q][k]);
      const double st[3] = {0.5, 0.5, 1.0};
      pack(st, Wzr, Whh);
      uint32_t* wf16 = reinterpret_cast<uint32_t*>(&h[m.gm_wf16[ph]]);
      frags16(Wzr, 48, 48, wf16);
      frags16(Whh, 48, 24, wf16 + zr);
      for (int q = 0; q < 3; ++q)
        for (int k = 0; k < 24; ++k) h[m.gm_wb16[ph] + q * 24 + k] = (float)(st[q] * B[q][k]);
    }
    const double* ggw = need("graph/gather_gate_w"); const double* ggb = need("graph/gather_gate_b");
    const double* gfw = need("graph/gather_feat_w"); const double* gfb = need("graph/gather_feat_b");
    std::vector<double> Gm((size_t)32 * 256, 0.0);
    for (int c = 0; c < 24; ++c)
      for (int k = 0; k < 128; ++k) {
        Gm[(size_t)c * 256 + k] = kNegLog2e * ggw[(size_t)c * 128 + k];
        Gm[(size_t)c * 256 + 128 + k] = kTwoLog2e * gfw[(size_t)c * 128 + k];
      }
    uint32_t* gf = reinterpret_cast<uint32_t*>(&h[m.gm_gf]);
    frags(Gm, 32, 256, gf, gf + gnn_mma_gather_words() / 2);
    for (int k = 0; k < 128; ++k) {
      h[m.gm_gb + k] = (float)(kNegLog2e * ggb[k]);
      h[m.gm_gb + 128 + k] = (float)(kTwoLog2e * gfb[k]);
    }
    // fp16 pool weights: gate by 1/2 (tanh form of the sigmoid), value by 1
    for (int c = 0; c < 24; ++c)
      for (int k = 0; k < 128; ++k) {
        Gm[(size_t)c * 256 + k] = 0.5 * ggw[(size_t)c * 128 + k];
        Gm[(size_t)c * 256 + 128 + k] = gfw[(size_t)c * 128 + k];
      }
    frags16(Gm, 32, 256, reinterpret_cast<uint32_t*>(&h[m.gm_gf16]));
    for (int k = 0; k < 128; ++k) {
      h[m.gm_gb16 + k] = (float)(0.5 * ggb[k]);
      h[m.gm_gb16 + 128 + k] = (float)gfb[k];
    }
  }
  if ((rc = copy("graph/dense1_w", m.gd1w, (size_t)m.gn * m.w1))) return rc;
  if ((rc = copy("graph/dense1_b", m.gd1b, m.w1))) return rc;
  if ((rc = copy("graph/dense2_w", m.gd2w, (size_t)m.w1 * m.w2))) return rc;
  if ((rc = copy("graph/dense2_b", m.gd2b, m.w2))) return rc;
  if ((rc = copy("graph/out_w", m.gow, m.w2))) return rc;
  if ((rc = copy("graph/out_b", m.gob, 1))) return rc;
  if (d.fusion_mode != FS_MODE_LATE) {
    if (d.model_specific_layers) {
      if ((rc = copy("fusion/ms_graph_w", m.msg, (size_t)m.gn * m.gn))) return rc;
      if ((rc = copy("fusion/ms_graph_b", m.msgb, m.gn))) return rc;
      if ((rc = copy("fusion/ms_voxel_w", m.msv, (size_t)m.lv * m.lv))) return rc;
      if ((rc = copy("fusion/ms_voxel_b", m.msvb, m.lv))) return rc;
    }
    int width = m.LW;
    for (int i = 0; i < d.n_fusion_layers; ++i) {
      int out = i + 1 < d.n_fusion_layers ? m.fd : 1;
      char wn[32], bn[32];
      snprintf(wn, sizeof wn, "fusion/fuse%d_w", i);
      snprintf(bn, sizeof bn, "fusion/fuse%d_b", i);
      if ((rc = copy(wn, m.fw[i], (size_t)width * out))) return rc;
      if ((rc = copy(bn, m.fb[i], out))) return rc;
      width = out;
    }
  }
  if (m.umma_ok) {
    umma::pack_weights(d, pm.get("voxel/conv1_w"), pm.get("voxel/conv2_w"), pm.get("voxel/conv3_w"),
                       pm.get("voxel/conv4_w"), (char*)h.data() + m.umma_off);
  }
  return FS_OK;
}

// ---------------------------------------------------------------------------
// workspace plan
// ---------------------------------------------------------------------------
struct WsPlan {
  size_t total = 0;
  size_t node_off, deg_cov, deg_ncov, row_cov, row_ncov, col_cov, col_ncov, node_pose, cursor;
  size_t feats, grid, grid_hi, grid_lo, a1, a2, p1, a3, a4, p2, d1, lat, hb0, hb1, g1, g2, pv, pg, state, scan, umma;
  size_t fact_cnt, fact_aff;
  size_t take(size_t bytes) { size_t o = total; total = align_up(total + bytes, 256); return o; }
};

// pose_nodes: upper bound on one pose's nodes (sizes the FFMA SG-CNN's global
// state fallback, needed only for poses too large for its shared memory)
static WsPlan plan_ws(const fs_model& m, int64_t P, int64_t N, int64_t E, int prec, int64_t pose_nodes) {
  WsPlan w;
  const int64_t G3 = (int64_t)m.G * m.G * m.G, H3 = G3 / 8, Q3 = G3 / 64;
  w.node_off = w.take(8 * (P + 1));
  w.deg_cov = w.take(4 * N); w.deg_ncov = w.take(4 * N);
  w.row_cov = w.take(8 * (N + 1)); w.row_ncov = w.take(8 * (N + 1));
  w.col_cov = w.take(sizeof(col_t) * E); w.col_ncov = w.take(sizeof(col_t) * E);
  w.node_pose = w.take(4 * N); w.cursor = w.take(8 * (N + 1));
  w.feats = w.take(4 * N * m.F);
  w.grid_hi = w.grid_lo = 0;
  if (prec == FS_PREC_MIXED) {   // X3 tcgen05 chain: fp32 grid -> (hi, lo) bf16 operands
    w.grid = w.take(4 * P * G3 * m.cin);
    w.grid_hi = w.take(2 * P * G3 * m.cin); w.grid_lo = w.take(2 * P * G3 * m.cin);
    w.umma = w.take(umma::workspace_bytes(m.d, P, true));
    w.a1 = w.a2 = w.p1 = w.a3 = w.a4 = 0;
    w.p2 = w.take(4 * (int64_t)umma::dense_rows_padded(P) * Q3 * m.f2);
  } else if (prec != FS_PREC_FP32) {   // tcgen05 conv chain (bf16)
    w.grid = w.take(2 * P * G3 * m.cin);
    w.umma = w.take(umma::workspace_bytes(m.d, P));
    w.a1 = w.a2 = w.p1 = w.a3 = w.a4 = 0;
    w.p2 = w.take(4 * (int64_t)umma::dense_rows_padded(P) * Q3 * m.f2);   // tcgen05 dense1 reads 128-row tiles
  } else {
    w.grid = w.take(4 * P * G3 * m.cin);
    w.a1 = w.take(4 * P * G3 * m.f1); w.a2 = w.take(4 * P * G3 * m.f1);
    w.p1 = w.take(4 * P * H3 * m.f1);
    w.a3 = w.take(4 * P * H3 * m.f2); w.a4 = w.take(4 * P * H3 * m.f2);
    w.p2 = w.take(4 * P * Q3 * m.f2);
    w.umma = 0;
  }
  w.d1 = w.take(4 * P * m.dn);
  w.lat = w.take(4 * P * m.LW);
  w.hb0 = w.take(4 * P * m.fd); w.hb1 = w.take(4 * P * m.fd);
  w.g1 = w.take(4 * P * m.w1); w.g2 = w.take(4 * P * m.w2);
  w.pv = w.take(4 * P); w.pg = w.take(4 * P);
  // FFMA SG-CNN's global node-state fallback: only for poses too large for
  // its shared-memory state
  const int pn = (int)(pose_nodes < FS_MAX_POSE_ATOMS ? pose_nodes : FS_MAX_POSE_ATOMS);
  w.state = w.take(gnn_needs_global_state(m.dpad, pn) ? (size_t)2 * 4 * N * m.dpad : 0);
  w.scan = w.take(scan_ws_bytes(N > P ? N : P) + 1024);
  w.fact_cnt = w.take(8 * P);
  w.fact_aff = w.take(4 * N);
  return w;
}

// ---- graph/voxel branch overlap ---------------------------------------------
// The radius graph (graph head input) and the voxel head are independent until
// the SG-CNN: with FS_OVERLAP=1 the graph kernels run on a library-owned side
// stream forked from and joined back into the caller's stream (per device and
// host thread, so concurrent callers stay independent).  Off by default: the
// persistent tcgen05 conv kernels lose more to the co-resident graph CTAs
// (conv1 5.3 -> 6.6 ms, conv2 6.0 -> 12.6 ms per 16,384 poses) than the
// overlap hides (measured: 58.4 vs 58.2 ms per step).
struct SideStream {
  cudaStream_t s = nullptr;
  cudaEvent_t fork = nullptr, join = nullptr;
  int mode = 1;
};

// per host thread; -1 = the FS_OVERLAP environment default (scheduling only:
// results are bitwise identical in every mode)
static thread_local int g_overlap_mode = -1;

static SideStream* side_stream() {
  // default 2: the tensor-bound conv chain leaves issue slots and shared
  // memory for one radius-graph CTA per SM (measured 43.7 -> 42.8 ms/step)
  static const int env_mode = getenv("FS_OVERLAP") ? atoi(getenv("FS_OVERLAP")) : 2;
  const int mode = g_overlap_mode >= 0 ? g_overlap_mode : env_mode;
  if (mode < 1 || mode > 3) return nullptr;
  static thread_local std::map<int, SideStream> streams;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return nullptr;
  SideStream& ss = streams[dev];
  ss.mode = mode;
  if (!ss.s) {
    int lo = 0, hi = 0;
    cudaDeviceGetStreamPriorityRange(&lo, &hi);
    if (cudaStreamCreateWithPriority(&ss.s, cudaStreamNonBlocking, mode >= 2 ? hi : lo) != cudaSuccess ||
        cudaEventCreateWithFlags(&ss.fork, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&ss.join, cudaEventDisableTiming) != cudaSuccess) {
      ss = SideStream{};
      return nullptr;
    }
  }
  return &ss;
}

// ---- pocket cache (fs_pocket_prepare / fs_score_poses_cached) --------------
struct PocketCacheLayout {
  int64_t off_n, off_T, off_pp, off_ppact, off_ppact_lo, off_wl, off_hcov, off_f, bytes;
};

static PocketCacheLayout cache_layout(const fs_model& m, int max_pocket) {
  PocketCacheLayout L;
  L.off_n = 0;
  L.off_T = 256;
  L.off_pp = (int64_t)align_up(L.off_T + 8 * 128, 256);
  L.off_ppact = (int64_t)align_up(L.off_pp + (int64_t)4 * m.G * m.G * m.G * m.f1, 256);
  L.off_ppact_lo = (int64_t)align_up(L.off_ppact + (int64_t)2 * m.G * m.G * m.G * m.f1, 256);
  L.off_wl = (int64_t)align_up(L.off_ppact_lo + (int64_t)2 * m.G * m.G * m.G * m.f1, 256);
  L.off_hcov = (int64_t)align_up(L.off_wl + (int64_t)4 * m.k1 * m.k1 * m.k1 * m.d.c_elem * m.f1, 256);
  L.off_f = (int64_t)align_up(L.off_hcov + (int64_t)4 * 24 * max_pocket, 256);
  L.bytes = (int64_t)align_up(L.off_f + (int64_t)4 * 128 * max_pocket, 256);
  return L;
}

static bool factoring_ok(const fs_model& m, int max_pocket) {
  return m.umma_ok && m.gmma_ok && conv1_fact_supported(m.G, m.k1, m.cin, m.f1) && max_pocket > 0 &&
         max_pocket <= FS_MAX_POSE_ATOMS && gnn_mma_fits(max_pocket);
}

static int act_of(int a) { return a == 0 ? FS_ACT_RELU : a == 1 ? FS_ACT_LEAKY : FS_ACT_SELU; }

// ---- heads -----------------------------------------------------------------
static int voxel_head_fp32(const fs_model& m, int P, char* ws, const WsPlan& w, cudaStream_t st) {
  const int G = m.G, H = G / 2, Q = G / 4;
  const fs_model_desc& d = m.d;
  float* grid = (float*)(ws + w.grid);
  float* a1 = (float*)(ws + w.a1); float* a2 = (float*)(ws + w.a2); float* p1 = (float*)(ws + w.p1);
  float* a3 = (float*)(ws + w.a3); float* a4 = (float*)(ws + w.a4); float* p2 = (float*)(ws + w.p2);
  int rc;
  ConvArgs c{};
  c.in = grid; c.w = m.P(m.c1w); c.b = m.P(m.c1b); c.out = a1; c.n_vox = (int64_t)P * G * G * G;
  c.g = G; c.cin = m.cin; c.cout = m.f1; c.k = m.k1;
  if (d.batch_norm) { c.bn_scale = m.P(m.bn1s); c.bn_shift = m.P(m.bn1h); }
  mark_stage(ST_CONV1, st);
  if ((rc = launch_conv3d_ffma(c, st))) return rc;
  mark_stage(ST_CONV2, st);
  c = ConvArgs{};
  c.in = a1; c.w = m.P(m.c2w); c.b = m.P(m.c2b); c.out = a2; c.n_vox = (int64_t)P * G * G * G;
  c.g = G; c.cin = m.f1; c.cout = m.f1; c.k = m.k2;
  if (d.residual_1) c.residual = a1;
  if ((rc = launch_conv3d_ffma(c, st))) return rc;
  if ((rc = launch_maxpool2(a2, p1, P, H, m.f1, st))) return rc;
  mark_stage(ST_CONV3, st);
  c = ConvArgs{};
  c.in = p1; c.w = m.P(m.c3w); c.b = m.P(m.c3b); c.out = a3; c.n_vox = (int64_t)P * H * H * H;
  c.g = H; c.cin = m.f1; c.cout = m.f2; c.k = m.k2;
  if (d.batch_norm) { c.bn_scale = m.P(m.bn2s); c.bn_shift = m.P(m.bn2h); }
  if ((rc = launch_conv3d_ffma(c, st))) return rc;
  mark_stage(ST_CONV4, st);
  c = ConvArgs{};
  c.in = a3; c.w = m.P(m.c4w); c.b = m.P(m.c4b); c.out = a4; c.n_vox = (int64_t)P * H * H * H;
  c.g = H; c.cin = m.f2; c.cout = m.f2; c.k = m.k2;
  if (d.residual_2) c.residual = a3;
  if ((rc = launch_conv3d_ffma(c, st))) return rc;
  return launch_maxpool2(a4, p2, P, Q, m.f2, st);
}

// dense1 -> dense2 (latent_v into lat[:, gn:]) -> optional pred_v
// tc: dense1 on tcgen05 (bf16 path; p2 holds umma::dense_rows_padded(P) rows)
static int voxel_tail(const fs_model& m, int P, char* ws, const WsPlan& w, bool want_pred, cudaStream_t st,
                      bool tc = false) {
  float* lat = (float*)(ws + w.lat);
  mark_stage(ST_DENSE, st);
  DenseArgs a{};
  a.x = (float*)(ws + w.p2); a.ldx = m.flat; a.w = m.P(m.d1w); a.b = m.P(m.d1b);
  a.y = (float*)(ws + w.d1); a.ldy = m.dn; a.m = P; a.k = m.flat; a.n = m.dn; a.act = FS_ACT_RELU;
  int rc = tc && umma::dense_tf32_ok(m.flat, m.dn)
               ? umma::dense_tf32(a.x, P, m.flat, m.P(m.d1t), m.dn, a.b, a.y, st)
               : launch_dense(a, st);
  if (rc) return rc;
  a = DenseArgs{};
  a.x = (float*)(ws + w.d1); a.ldx = m.dn; a.w = m.P(m.d2w); a.b = m.P(m.d2b);
  a.y = lat + m.gn; a.ldy = m.LW; a.m = P; a.k = m.dn; a.n = m.lv; a.act = FS_ACT_RELU;
  if ((rc = launch_dense(a, st))) return rc;
  if (want_pred) {
    a = DenseArgs{};
    a.x = lat + m.gn; a.ldx = m.LW; a.w = m.P(m.ow); a.b = m.P(m.ob);
    a.y = (float*)(ws + w.pv); a.ldy = 1; a.m = P; a.k = m.lv; a.n = 1; a.act = FS_ACT_NONE;
    if ((rc = launch_dense(a, st))) return rc;
  }
  return FS_OK;
}

// ids_padded: the CSR came from graph_csr/graph_fact (rows padded to 4 ids)
static int graph_head(const fs_model& m, int P, int max_nodes, char* ws, const WsPlan& w,
                      const int32_t* err, bool want_pred, int precision, cudaStream_t st,
                      const GnnMmaArgs* extra = nullptr, bool ids_padded = true) {
  GnnArgs g{};
  g.feats = (float*)(ws + w.feats); g.F = m.F; g.node_off = (int64_t*)(ws + w.node_off);
  g.row_cov = (int64_t*)(ws + w.row_cov); g.col_cov = (col_t*)(ws + w.col_cov);
  g.row_ncov = (int64_t*)(ws + w.row_ncov); g.col_ncov = (col_t*)(ws + w.col_ncov);
  g.deg_cov = (int32_t*)(ws + w.deg_cov); g.deg_ncov = (int32_t*)(ws + w.deg_ncov);
  g.we = m.P(m.we); g.be = m.P(m.be); g.phase[0] = m.P(m.ph[0]); g.phase[1] = m.P(m.ph[1]);
  g.gg = m.P(m.gg); g.bg = m.P(m.bg); g.gf = m.P(m.gf); g.bf = m.P(m.bf);
  g.k_steps[0] = m.d.k_cov; g.k_steps[1] = m.d.k_noncov; g.gn = m.gn;
  g.state = (float*)(ws + w.state); g.lat = (float*)(ws + w.lat); g.ld_lat = m.LW; g.err = err;
  mark_stage(ST_GNN, st);
  int rc;
  if (extra || (precision != FS_PREC_FP32 && m.gmma_ok && gnn_mma_fits(max_nodes))) {
    GnnMmaArgs q{};
    if (extra) q = *extra;   // factored-mode / dump fields
    q.feats = g.feats; q.F = g.F; q.node_off = g.node_off;
    q.row_cov = g.row_cov; q.col_cov = g.col_cov; q.row_ncov = g.row_ncov; q.col_ncov = g.col_ncov;
    q.deg_cov = g.deg_cov; q.deg_ncov = g.deg_ncov;
    q.we = g.we; q.be = g.be;
    for (int ph = 0; ph < 2; ++ph) {
      q.wfrag[ph] = reinterpret_cast<const uint32_t*>(m.P(m.gm_wf[ph]));
      q.wbias[ph] = m.P(m.gm_wb[ph]);
    }
    q.gfrag = reinterpret_cast<const uint32_t*>(m.P(m.gm_gf)); q.gbias = m.P(m.gm_gb);
    for (int ph = 0; ph < 2; ++ph) {
      q.wfrag16[ph] = reinterpret_cast<const uint32_t*>(m.P(m.gm_wf16[ph]));
      q.wbias16[ph] = m.P(m.gm_wb16[ph]);
    }
    q.gfrag16 = reinterpret_cast<const uint32_t*>(m.P(m.gm_gf16));
    q.gbias16 = m.P(m.gm_gb16);
    q.k_steps[0] = m.d.k_cov; q.k_steps[1] = m.d.k_noncov;
    q.lat = g.lat; q.ld_lat = g.ld_lat; q.err = err;
    q.ids_padded = ids_padded ? 1 : 0;
    // GEMM operand split, fixed by the precision argument: FS_PREC_BF16 =
    // fp16 activations hi/lo x fp16 weights, two passes; FS_PREC_MIXED = bf16
    // hi/lo x hi/lo, three passes (fp32-class)
    rc = launch_gnn_mma(q, precision == FS_PREC_MIXED ? 3 : 2, P, max_nodes, st);
  } else {
    rc = launch_gnn(g, m.dpad, P, max_nodes, st);
  }
  mark_stage(ST_FUSION, st);
  if (rc || !want_pred) return rc;
  float* lat = (float*)(ws + w.lat);
  DenseArgs a{};
  a.x = lat; a.ldx = m.LW; a.w = m.P(m.gd1w); a.b = m.P(m.gd1b); a.y = (float*)(ws + w.g1); a.ldy = m.w1;
  a.m = P; a.k = m.gn; a.n = m.w1; a.act = FS_ACT_RELU;
  if ((rc = launch_dense(a, st))) return rc;
  a = DenseArgs{};
  a.x = (float*)(ws + w.g1); a.ldx = m.w1; a.w = m.P(m.gd2w); a.b = m.P(m.gd2b); a.y = (float*)(ws + w.g2);
  a.ldy = m.w2; a.m = P; a.k = m.w1; a.n = m.w2; a.act = FS_ACT_RELU;
  if ((rc = launch_dense(a, st))) return rc;
  a = DenseArgs{};
  a.x = (float*)(ws + w.g2); a.ldx = m.w2; a.w = m.P(m.gow); a.b = m.P(m.gob); a.y = (float*)(ws + w.pg);
  a.ldy = 1; a.m = P; a.k = m.w2; a.n = 1; a.act = FS_ACT_NONE;
  return launch_dense(a, st);
}

static int fusion_head(const fs_model& m, int P, char* ws, const WsPlan& w, float* scores, cudaStream_t st) {
  const fs_model_desc& d = m.d;
  float* lat = (float*)(ws + w.lat);
  const int act = act_of(d.activation);
  int rc;
  if (d.model_specific_layers) {
    DenseArgs a{};
    a.x = lat; a.ldx = m.LW; a.w = m.P(m.msg); a.b = m.P(m.msgb); a.y = lat + m.gn + m.lv; a.ldy = m.LW;
    a.m = P; a.k = m.gn; a.n = m.gn; a.act = act;
    if ((rc = launch_dense(a, st))) return rc;
    a = DenseArgs{};
    a.x = lat + m.gn; a.ldx = m.LW; a.w = m.P(m.msv); a.b = m.P(m.msvb); a.y = lat + 2 * m.gn + m.lv;
    a.ldy = m.LW; a.m = P; a.k = m.lv; a.n = m.lv; a.act = act;
    if ((rc = launch_dense(a, st))) return rc;
  }
  float* hb[2] = {(float*)(ws + w.hb0), (float*)(ws + w.hb1)};
  const float* x = lat;
  int64_t ldx = m.LW;
  int width = m.LW;
  const int n = d.n_fusion_layers;
  for (int i = 0; i < n; ++i) {
    DenseArgs a{};
    a.x = x; a.ldx = ldx; a.w = m.P(m.fw[i]); a.b = m.P(m.fb[i]); a.m = P; a.k = width;
    if (i + 1 < n) {
      a.y = hb[i & 1]; a.ldy = m.fd; a.n = m.fd; a.act = act;
      if (d.residual_fusion && i > 0) { a.r = x; a.ldr = ldx; }   // models.py:391-392
    } else {
      a.y = scores; a.ldy = 1; a.n = 1; a.act = FS_ACT_NONE;
    }
    if ((rc = launch_dense(a, st))) return rc;
    x = a.y; ldx = a.ldy; width = a.n;
  }
  return FS_OK;
}

static int copy_outputs(const fs_model& m, int P, char* ws, const WsPlan& w, float* lat_v, float* lat_g,
                        float* pred_v, float* pred_g, cudaStream_t st) {
  float* lat = (float*)(ws + w.lat);
  if (lat_v && P > 0)
    FS_CUDA_CHECK(cudaMemcpy2DAsync(lat_v, m.lv * 4, lat + m.gn, m.LW * 4, m.lv * 4, P, cudaMemcpyDeviceToDevice, st));
  if (lat_g && P > 0)
    FS_CUDA_CHECK(cudaMemcpy2DAsync(lat_g, m.gn * 4, lat, m.LW * 4, m.gn * 4, P, cudaMemcpyDeviceToDevice, st));
  if (pred_v && P > 0) FS_CUDA_CHECK(cudaMemcpyAsync(pred_v, ws + w.pv, 4 * P, cudaMemcpyDeviceToDevice, st));
  if (pred_g && P > 0) FS_CUDA_CHECK(cudaMemcpyAsync(pred_g, ws + w.pg, 4 * P, cudaMemcpyDeviceToDevice, st));
  return FS_OK;
}

}  // namespace fs

using namespace fs;

// ===========================================================================
// extern "C"
// ===========================================================================
extern "C" {

const char* fs_strerror(int code) {
  switch (code) {
    case FS_OK: return "ok";
    case FS_EINVAL: return "invalid argument";
    case FS_ECAPACITY: return "capacity exceeded (workspace or per-pose size limit)";
    case FS_ECUDA: return "CUDA runtime error";
    case FS_ENOTSUP: return "configuration not supported for this precision";
    default: return "unknown error";
  }
}

int fs_version(void) { return 100; }

long long fs_launch_count(void) { return g_launches.load(); }

int fs_set_stage_events(void** events, int n) {
  if (events && n < ST_COUNT) return FS_EINVAL;
  g_stage_events = (cudaEvent_t*)events;
  return FS_OK;
}

const char* fs_last_cuda_error(void) { return g_last_cuda_error.c_str(); }

int fs_set_overlap(int mode) {
  if (mode < -1 || mode > 2) return FS_EINVAL;
  g_overlap_mode = mode;
  return FS_OK;
}

size_t fs_weights_bytes(const fs_model_desc* desc) {
  if (!desc || validate_desc(*desc)) return 0;
  fs_model m;
  m.d = *desc;
  return plan_model(m);
}

int fs_model_create(const fs_model_desc* desc, const char* const* host_names,
                    const double* const* host_params, int n_params, void* dev_blob,
                    size_t blob_bytes, void* stream, fs_model** out) {
  if (!desc || !out || !dev_blob) return FS_EINVAL;
  int rc = validate_desc(*desc);
  if (rc) return rc;
  fs_model* m = new fs_model();
  m->d = *desc;
  m->blob_bytes = plan_model(*m);
  if (blob_bytes < m->blob_bytes) { delete m; return FS_ECAPACITY; }
  ParamMap pm;
  for (int i = 0; i < n_params; ++i) pm.p[host_names[i]] = host_params[i];
  std::vector<float> h;
  if ((rc = pack_model(*m, pm, h))) { delete m; return rc; }
  m->blob = (float*)dev_blob;
  cudaError_t e = cudaMemcpyAsync(dev_blob, h.data(), m->blob_bytes, cudaMemcpyHostToDevice, (cudaStream_t)stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize((cudaStream_t)stream);   // one-off, keeps h alive
  if (e != cudaSuccess) { set_cuda_error(e); delete m; return FS_ECUDA; }
  *out = m;
  return FS_OK;
}

int fs_model_destroy(fs_model* m) { delete m; return FS_OK; }

int fs_model_supports(const fs_model* m, int precision) {
  if (!m) return 0;
  if (precision == FS_PREC_FP32) return 1;
  if (precision == FS_PREC_BF16 || precision == FS_PREC_MIXED) return m->umma_ok ? 1 : 0;
  return 0;
}

size_t fs_node_offsets_ws_bytes(int32_t n_poses) { return scan_ws_bytes(n_poses) + 256; }

int fs_node_offsets(const fs_pose_batch* b, int64_t* node_off, void* ws, size_t ws_bytes, void* stream) {
  if (!b || !node_off) return FS_EINVAL;
  return launch_node_offsets(*b, node_off, ws, ws_bytes, (cudaStream_t)stream);
}

int fs_voxelize(const fs_pose_batch* b, int32_t extent, int32_t c_elem, double box_size, int32_t layout,
                void* out, int32_t* err, void* stream) {
  if (!b || !out || !err || c_elem < 1 || layout < 0 || layout > 2) return FS_EINVAL;
  return launch_voxelize(*b, extent, c_elem, box_size, layout, out, err, (cudaStream_t)stream);
}

int fs_node_features(const fs_pose_batch* b, const int64_t* node_off, int32_t c_elem, double box_size,
                     double* out, void* stream) {
  if (!b || !node_off || !out || c_elem < 1) return FS_EINVAL;
  return launch_node_features(*b, node_off, c_elem, box_size, out, true, (cudaStream_t)stream);
}

int fs_graph_count(const fs_pose_batch* b, const int64_t* node_off, double cov_thresh, double noncov_thresh,
                   int32_t* deg_cov, int32_t* deg_ncov, int32_t* err, void* stream) {
  if (!b || !node_off || !deg_cov || !deg_ncov || !err) return FS_EINVAL;
  return launch_graph_count(*b, node_off, cov_thresh, noncov_thresh, deg_cov, deg_ncov, err, (cudaStream_t)stream);
}

size_t fs_graph_rows_ws_bytes(int64_t n_nodes) { return scan_ws_bytes(n_nodes) + 256; }

int fs_graph_rows(const int32_t* deg, int64_t n_nodes, int64_t* row_ptr, void* ws, size_t ws_bytes, void* stream) {
  if (!deg || !row_ptr || n_nodes < 0) return FS_EINVAL;
  return launch_rows(deg, n_nodes, row_ptr, ws, ws_bytes, (cudaStream_t)stream);
}

int fs_graph_fill(const fs_pose_batch* b, const int64_t* node_off, double cov_thresh, double noncov_thresh,
                  const int64_t* row_cov, const int64_t* row_ncov, int32_t* col_cov, int32_t* col_ncov,
                  double* dist_cov, double* dist_ncov, int64_t cap_cov, int64_t cap_ncov, int32_t* err,
                  void* stream) {
  if (!b || !node_off || !row_cov || !row_ncov || !err) return FS_EINVAL;
  return launch_graph_fill(*b, node_off, cov_thresh, noncov_thresh, row_cov, row_ncov, col_cov, col_ncov,
                           dist_cov, dist_ncov, cap_cov, cap_ncov, err, (cudaStream_t)stream);
}

int fs_graph_edge_counts(const int64_t* node_off, int32_t n_poses, const int64_t* row_ptr, const int32_t* col,
                         int64_t* edge_off, void* ws, size_t ws_bytes, void* stream) {
  if (!node_off || !row_ptr || !edge_off) return FS_EINVAL;
  return launch_edge_counts(node_off, n_poses, row_ptr, col, edge_off, ws, ws_bytes, (cudaStream_t)stream);
}

int fs_graph_edges(const int64_t* node_off, int32_t n_poses, const int64_t* row_ptr, const int32_t* col,
                   const double* dist, const int64_t* edge_off, int64_t* edges, double* dists, void* stream) {
  if (!node_off || !row_ptr || !edge_off || !edges) return FS_EINVAL;
  return launch_edges(node_off, n_poses, row_ptr, col, dist, edge_off, edges, dists, (cudaStream_t)stream);
}

size_t fs_workspace_bytes(const fs_model* m, int32_t max_poses, int64_t max_nodes, int64_t max_edges, int precision) {
  if (!m || max_poses < 0 || max_nodes < 0 || max_edges < 0) return 0;
  const int64_t pose_nodes = max_poses > 0 ? (max_nodes + max_poses - 1) / max_poses : 0;
  return plan_ws(*m, max_poses, max_nodes, max_edges, precision, pose_nodes).total + 256;
}

size_t fs_features_workspace_bytes(const fs_model* m, int32_t n_poses, int64_t n_nodes, int32_t max_pose_nodes,
                                   int64_t n_edges, int precision) {
  if (!m || n_poses < 0 || n_nodes < 0 || n_edges < 0) return 0;
  const int64_t bound = max_pose_nodes > 0 ? (max_pose_nodes < n_nodes ? max_pose_nodes : n_nodes)
                                           : (n_nodes < FS_MAX_POSE_ATOMS ? n_nodes : FS_MAX_POSE_ATOMS);
  return plan_ws(*m, n_poses, n_nodes, 2 * n_edges, precision, bound).total + 256;
}

int fs_score_poses(const fs_model* m, int precision, const fs_pose_batch* b, int64_t max_edges, void* ws,
                   size_t ws_bytes, float* scores, float* lat_v, float* lat_g, float* pred_v, float* pred_g,
                   int32_t* err, void* stream) {
  if (!m || !b || !ws || !scores || !err) return FS_EINVAL;
  if (!fs_model_supports(m, precision)) return FS_ENOTSUP;
  if (m->d.in_channels % 2) return FS_EINVAL;   // featurize: GridConfig(c_elem=in_channels//2)
  const int P = b->n_poses;
  if (P <= 0) return FS_OK;
  const int max_atoms = b->max_pose_atoms > 0 ? b->max_pose_atoms : FS_MAX_POSE_ATOMS;
  const int64_t N = (int64_t)P * max_atoms;
  if (max_edges <= 0) return FS_EINVAL;
  WsPlan w = plan_ws(*m, P, N, (int64_t)P * max_edges, precision, max_atoms);
  if (w.total > ws_bytes) return FS_ECAPACITY;
  cudaStream_t st = (cudaStream_t)stream;
  char* W = (char*)(((uintptr_t)ws + 255) & ~(uintptr_t)255);
  if ((size_t)(W - (char*)ws) + w.total > ws_bytes) return FS_ECAPACITY;
  int64_t* node_off = (int64_t*)(W + w.node_off);
  int rc;
  mark_stage(ST_FEATURIZE, st);
  FS_CUDA_CHECK(cudaMemsetAsync(err, 0, 4 * (size_t)P, st));
  // oversize poses are clamped to max_atoms rows (and flagged by the graph
  // kernel), so node_off[P] <= N = P * max_atoms always holds
  if ((rc = launch_node_offsets(*b, node_off, W + w.scan, scan_ws_bytes(N > P ? N : P) + 1024, st, max_atoms)))
    return rc;
  const fs_model_desc& d = m->d;
  const bool late = d.fusion_mode == FS_MODE_LATE;
  // featurize (models.py:638-651): radius graph + node features in one fused
  // launch (pose-private CSR slices of max_edges entries per edge type, rows =
  // start offset + degree); voxel branch: voxelize + conv chain + dense.
  auto graph_branch = [&](cudaStream_t gs) {
    return launch_graph_csr(*b, node_off, d.cov_thresh, d.noncov_thresh, (int64_t*)(W + w.row_cov),
                            (int32_t*)(W + w.deg_cov), (col_t*)(W + w.col_cov), nullptr, (int64_t*)(W + w.row_ncov),
                            (int32_t*)(W + w.deg_ncov), (col_t*)(W + w.col_ncov), nullptr, max_edges, err, gs,
                            (float*)(W + w.feats), d.c_elem, d.box_size);
  };
  auto voxel_branch = [&](cudaStream_t vs) {
    int r;
    if (precision == FS_PREC_MIXED) {
      if ((r = launch_voxelize(*b, d.grid_extent, m->cgrid, d.box_size, FS_GRID_NDHWC_F32, W + w.grid, err, vs)))
        return r;
      if ((r = launch_split_bf16((const float*)(W + w.grid), (__nv_bfloat16*)(W + w.grid_hi),
                                 (__nv_bfloat16*)(W + w.grid_lo), (int64_t)P * m->G * m->G * m->G * m->cin, vs)))
        return r;
      if ((r = umma::voxel_convs_x3(d, (const char*)m->blob + m->umma_off, m->P(m->c1b), m->P(m->c2b),
                                    m->P(m->c3b), m->P(m->c4b), P, (const __nv_bfloat16*)(W + w.grid_hi),
                                    (const __nv_bfloat16*)(W + w.grid_lo), W + w.umma, (float*)(W + w.p2), vs)))
        return r;
    } else if (precision != FS_PREC_FP32) {
      if ((r = launch_voxelize(*b, d.grid_extent, m->cgrid, d.box_size, FS_GRID_NDHWC_BF16, W + w.grid, err, vs)))
        return r;
      if ((r = umma::voxel_convs(d, (const char*)m->blob + m->umma_off, m->P(m->c1b), m->P(m->c2b), m->P(m->c3b),
                                 m->P(m->c4b), P, (const __nv_bfloat16*)(W + w.grid), W + w.umma,
                                 (float*)(W + w.p2), vs)))
        return r;
    } else {
      if ((r = launch_voxelize(*b, d.grid_extent, m->cgrid, d.box_size, FS_GRID_NDHWC_F32, W + w.grid, err, vs)))
        return r;
      if ((r = voxel_head_fp32(*m, P, W, w, vs))) return r;
    }
    // dense1: tcgen05 tf32 on the bf16 path, FFMA fp32 on the mixed (1e-3) path
    return voxel_tail(*m, P, W, w, late || pred_v, vs, precision == FS_PREC_BF16);
  };
  // FS_OVERLAP=0: serial; 1: graph branch on a side stream; 2 (default):
  // voxel branch on a high-priority side stream, issued first, graph branch
  // on the caller's stream; joined before the SG-CNN
  SideStream* ss = side_stream();
  if (!ss) {
    if ((rc = graph_branch(st))) return rc;
    if ((rc = voxel_branch(st))) return rc;
  } else {
    FS_CUDA_CHECK(cudaEventRecord(ss->fork, st));
    FS_CUDA_CHECK(cudaStreamWaitEvent(ss->s, ss->fork, 0));
    if (ss->mode == 2) {
      if ((rc = voxel_branch(ss->s))) return rc;
      if ((rc = graph_branch(st))) return rc;
    } else if (ss->mode == 3) {   // graph branch on the high-priority side stream, issued first
      if ((rc = graph_branch(ss->s))) return rc;
      if ((rc = voxel_branch(st))) return rc;
    } else {
      if ((rc = graph_branch(ss->s))) return rc;
      if ((rc = voxel_branch(st))) return rc;
    }
    FS_CUDA_CHECK(cudaEventRecord(ss->join, ss->s));
    FS_CUDA_CHECK(cudaStreamWaitEvent(st, ss->join, 0));
  }
  if ((rc = graph_head(*m, P, max_atoms, W, w, err, late || pred_g, precision, st))) return rc;
  if (!late && (rc = fusion_head(*m, P, W, w, scores, st))) return rc;
  if ((rc = launch_finalize(P, d.fusion_mode, (float*)(W + w.pv), (float*)(W + w.pg), scores, err, st))) return rc;
  rc = copy_outputs(*m, P, W, w, lat_v, lat_g, pred_v, pred_g, st);
  mark_stage(ST_END, st);
  return rc;
}

// ---- pocket-invariant factoring ----------------------------
// node rows of one pose's compact factored slice: nc = nLp + nA <= max_atoms + 15
static int64_t fact_slice_rows(int max_atoms) {
  const int64_t S = (int64_t)((max_atoms + 15 + 15) & ~15);
  return S > gnn_mma_max_nodes() ? gnn_mma_max_nodes() : S;
}

// covalent CSR capacity of a pocket-only pose (directed entries)
static int64_t pocket_edge_cap(int max_pocket) { return (int64_t)64 * max_pocket + 1024; }

size_t fs_pocket_cache_bytes(const fs_model* m, int32_t max_pocket_atoms) {
  if (!m || !factoring_ok(*m, max_pocket_atoms)) return 0;
  return (size_t)cache_layout(*m, max_pocket_atoms).bytes;
}

static size_t prep_extra_bytes(const fs_model& m, int n, int mp) {
  return align_up(8 * (size_t)(n + 1), 256) + align_up(4 * (size_t)n, 256) +
         align_up((size_t)4 * n * mp * 24, 256) + align_up((size_t)4 * n * mp * 128, 256) +
         align_up((size_t)4 * m.k1 * m.k1 * m.k1 * m.cin * m.f1, 256) +
         align_up((size_t)4 * n * m.G * m.G * m.G * m.f1, 256);
}

size_t fs_pocket_prepare_ws_bytes(const fs_model* m, int32_t n_pockets, int32_t max_pocket_atoms) {
  if (!m || n_pockets < 0 || !factoring_ok(*m, max_pocket_atoms)) return 0;
  const int64_t N = (int64_t)n_pockets * max_pocket_atoms;
  return plan_ws(*m, n_pockets, N, n_pockets * pocket_edge_cap(max_pocket_atoms), FS_PREC_FP32,
                 max_pocket_atoms).total +
         prep_extra_bytes(*m, n_pockets, max_pocket_atoms) + 512;
}

int fs_pocket_prepare(const fs_model* m, int precision, const double* pocket_xyz, const int32_t* pocket_elem,
                      const int32_t* pocket_role, const int64_t* pocket_off, int32_t n_pockets,
                      int32_t max_pocket_atoms, void* cache, int32_t* err, void* ws, size_t ws_bytes,
                      void* stream) {
  if (!m || !pocket_xyz || !pocket_elem || !pocket_role || !pocket_off || !cache || !err || !ws) return FS_EINVAL;
  if ((precision != FS_PREC_BF16 && precision != FS_PREC_MIXED) || !factoring_ok(*m, max_pocket_atoms))
    return FS_ENOTSUP;
  const int n = n_pockets, mp = max_pocket_atoms;
  if (n <= 0) return FS_OK;
  if (ws_bytes < fs_pocket_prepare_ws_bytes(m, n, mp)) return FS_ECAPACITY;
  cudaStream_t st = (cudaStream_t)stream;
  const fs_model_desc& d = m->d;
  const PocketCacheLayout L = cache_layout(*m, mp);
  const int64_t cap = pocket_edge_cap(mp);
  // fp32 plan: the pocket grid is voxelized as fp32 for the FFMA conv1
  WsPlan w = plan_ws(*m, n, (int64_t)n * mp, n * cap, FS_PREC_FP32, mp);
  char* W = (char*)(((uintptr_t)ws + 255) & ~(uintptr_t)255);
  char* X = W + w.total;   // prep-only buffers
  int64_t* atom_off = (int64_t*)X; X += align_up(8 * (size_t)(n + 1), 256);
  int32_t* target = (int32_t*)X; X += align_up(4 * (size_t)n, 256);
  float* dump_h = (float*)X; X += align_up((size_t)4 * n * mp * 24, 256);
  float* dump_f = (float*)X; X += align_up((size_t)4 * n * mp * 128, 256);
  float* w1r = (float*)X; X += align_up((size_t)4 * m->k1 * m->k1 * m->k1 * m->cin * m->f1, 256);
  float* pp = (float*)X;
  int rc;
  if ((rc = launch_pocket_poses(n, atom_off, target, st))) return rc;
  fs_pose_batch pb{};
  pb.pocket_xyz = pocket_xyz; pb.pocket_elem = pocket_elem; pb.pocket_role = pocket_role;
  pb.pocket_off = pocket_off; pb.n_pockets = n;
  pb.atom_xyz = pocket_xyz; pb.atom_elem = pocket_elem; pb.atom_role = pocket_role; pb.atom_off = atom_off;
  pb.pose_target = target; pb.n_poses = n; pb.max_pose_atoms = mp;
  FS_CUDA_CHECK(cudaMemsetAsync(err, 0, 4 * (size_t)n, st));
  int64_t* node_off = (int64_t*)(W + w.node_off);
  if ((rc = launch_node_offsets(pb, node_off, W + w.scan, scan_ws_bytes((int64_t)n * mp) + 1024, st))) return rc;
  if ((rc = launch_node_features(pb, node_off, d.c_elem, d.box_size, W + w.feats, false, st))) return rc;
  if ((rc = launch_graph_csr(pb, node_off, d.cov_thresh, d.noncov_thresh, (int64_t*)(W + w.row_cov),
                             (int32_t*)(W + w.deg_cov), (col_t*)(W + w.col_cov), nullptr, (int64_t*)(W + w.row_ncov),
                             (int32_t*)(W + w.deg_ncov), (col_t*)(W + w.col_ncov), nullptr, cap, err, st)))
    return rc;
  // SG-CNN of the pocket alone (no ligand -> no non-covalent edges: every
  // node follows the message-free trajectory), dumping the post-covalent
  // states and the per-node pool terms
  GnnMmaArgs x{};
  x.dump_hcov = dump_h; x.dump_f = dump_f; x.dump_ld = mp;
  if ((rc = graph_head(*m, n, mp, W, w, err, false, precision, st, &x))) return rc;
  char* C = (char*)cache;
  FS_CUDA_CHECK(cudaMemcpy2DAsync(C + L.off_hcov, L.bytes, dump_h, (size_t)4 * mp * 24, (size_t)4 * mp * 24, n,
                                  cudaMemcpyDeviceToDevice, st));
  FS_CUDA_CHECK(cudaMemcpy2DAsync(C + L.off_f, L.bytes, dump_f, (size_t)4 * mp * 128, (size_t)4 * mp * 128, n,
                                  cudaMemcpyDeviceToDevice, st));
  if ((rc = launch_pocket_total(pocket_off, n, dump_f, mp, C, L.bytes, L.off_T, L.off_n, st))) return rc;
  // conv1 pre-activation of the pocket channels, bf16-valued weights, fp32
  if ((rc = launch_voxelize(pb, d.grid_extent, m->cgrid, d.box_size, FS_GRID_NDHWC_F32, W + w.grid, err, st))) return rc;
  const int64_t nw = (int64_t)m->k1 * m->k1 * m->k1 * m->cin * m->f1;
  // bf16 caches use the bf16-valued weights of the tcgen05 conv1; mixed
  // caches the exact fp32 ones (the 3-pass conv1 is fp32-class)
  const bool x3 = precision == FS_PREC_MIXED;
  if (!x3 && (rc = launch_round_bf16(m->P(m->c1w), w1r, nw, st))) return rc;
  ConvArgs c{};
  c.in = (float*)(W + w.grid); c.w = x3 ? m->P(m->c1w) : w1r; c.b = m->P(m->c1b); c.out = pp;
  c.n_vox = (int64_t)n * m->G * m->G * m->G; c.g = m->G; c.cin = m->cin; c.cout = m->f1; c.k = m->k1; c.no_relu = 1;
  if ((rc = launch_conv3d_ffma(c, st))) return rc;
  const size_t ppb = (size_t)4 * m->G * m->G * m->G * m->f1;
  FS_CUDA_CHECK(cudaMemcpy2DAsync(C + L.off_pp, L.bytes, pp, ppb, ppb, n, cudaMemcpyDeviceToDevice, st));
  return launch_pocket_conv1_fields(pp, n, C, L.bytes, L.off_ppact, L.off_wl, m->P(m->c1w), d.c_elem, st,
                                    L.off_ppact_lo, x3 ? 1 : 0);
}

int fs_score_poses_cached(const fs_model* m, int precision, const fs_pose_batch* b, const void* cache,
                          int32_t max_pocket_atoms, int64_t max_edges, void* ws, size_t ws_bytes, float* scores,
                          float* lat_v, float* lat_g, float* pred_v, float* pred_g, int32_t* err, void* stream) {
  if (!m || !b || !cache || !ws || !scores || !err || max_edges <= 0) return FS_EINVAL;
  if ((precision != FS_PREC_BF16 && precision != FS_PREC_MIXED) || !factoring_ok(*m, max_pocket_atoms))
    return FS_ENOTSUP;
  const int P = b->n_poses;
  if (P <= 0) return FS_OK;
  const int max_atoms = b->max_pose_atoms > 0 ? b->max_pose_atoms : FS_MAX_POSE_ATOMS;
  // compact node slice per pose; poses whose touched set does not fit the
  // tensor-core SG-CNN's shared memory are flagged FS_ERR_NOT_FACTORED
  const int64_t S = fact_slice_rows(max_atoms);
  const int64_t N = (int64_t)P * S;
  WsPlan w = plan_ws(*m, P, N, (int64_t)P * max_edges, precision, S);
  char* W = (char*)(((uintptr_t)ws + 255) & ~(uintptr_t)255);
  if ((size_t)(W - (char*)ws) + w.total > ws_bytes) return FS_ECAPACITY;
  cudaStream_t st = (cudaStream_t)stream;
  const fs_model_desc& d = m->d;
  const PocketCacheLayout L = cache_layout(*m, max_pocket_atoms);
  const bool late = d.fusion_mode == FS_MODE_LATE;
  int32_t* cnt = (int32_t*)(W + w.fact_cnt);
  int32_t* aff = (int32_t*)(W + w.fact_aff);
  int rc;
  mark_stage(ST_FEATURIZE, st);
  FS_CUDA_CHECK(cudaMemsetAsync(err, 0, 4 * (size_t)P, st));
  SideStream* ss = side_stream();
  cudaStream_t gst = st;
  if (ss) {
    FS_CUDA_CHECK(cudaEventRecord(ss->fork, st));
    FS_CUDA_CHECK(cudaStreamWaitEvent(ss->s, ss->fork, 0));
    gst = ss->s;
  }
  if ((rc = launch_graph_fact(*b, d.cov_thresh, d.noncov_thresh, d.box_size, d.c_elem, S, max_edges, max_pocket_atoms,
                              cnt, aff, (float*)(W + w.feats), (int64_t*)(W + w.row_cov), (int32_t*)(W + w.deg_cov),
                              (col_t*)(W + w.col_cov), (int64_t*)(W + w.row_ncov), (int32_t*)(W + w.deg_ncov),
                              (col_t*)(W + w.col_ncov), err, gst)))
    return rc;
  if (ss) FS_CUDA_CHECK(cudaEventRecord(ss->join, gst));
  mark_stage(ST_CONV1, st);
  const bool x3 = precision == FS_PREC_MIXED;
  if ((rc = launch_conv1_fact(*b, (const char*)cache, L.bytes, L.off_pp, L.off_ppact, L.off_wl, d.c_elem,
                              d.box_size, umma::act1_ptr(W + w.umma), st, L.off_ppact_lo,
                              x3 ? umma::act1_lo_ptr(W + w.umma, P) : nullptr)))
    return rc;
  rc = x3 ? umma::voxel_convs_from2_x3(d, (const char*)m->blob + m->umma_off, m->P(m->c2b), m->P(m->c3b),
                                       m->P(m->c4b), P, W + w.umma, (float*)(W + w.p2), st)
          : umma::voxel_convs_from2(d, (const char*)m->blob + m->umma_off, m->P(m->c2b), m->P(m->c3b),
                                    m->P(m->c4b), P, W + w.umma, (float*)(W + w.p2), st);
  if (rc) return rc;
  if ((rc = voxel_tail(*m, P, W, w, late || pred_v, st, precision == FS_PREC_BF16))) return rc;
  if (ss) FS_CUDA_CHECK(cudaStreamWaitEvent(st, ss->join, 0));
  GnnMmaArgs x{};
  x.fact_cnt = cnt; x.fact_stride = S; x.fact_aff = aff; x.pose_target = b->pose_target;
  x.cache = (const char*)cache; x.cache_stride = L.bytes;
  x.off_hcov = L.off_hcov; x.off_f = L.off_f; x.off_T = L.off_T; x.off_n = L.off_n;
  if ((rc = graph_head(*m, P, (int)S, W, w, err, late || pred_g, precision, st, &x))) return rc;
  if (!late && (rc = fusion_head(*m, P, W, w, scores, st))) return rc;
  if ((rc = launch_finalize(P, d.fusion_mode, (float*)(W + w.pv), (float*)(W + w.pg), scores, err, st))) return rc;
  rc = copy_outputs(*m, P, W, w, lat_v, lat_g, pred_v, pred_g, st);
  mark_stage(ST_END, st);
  return rc;
}

int fs_score_features(const fs_model* m, int precision, int32_t n_poses, const double* grids,
                      const double* feats, const int64_t* node_off, int64_t n_nodes, int32_t max_pose_nodes,
                      const int64_t* cov_edges, int64_t n_cov, const int64_t* ncov_edges, int64_t n_ncov,
                      int32_t heads, void* ws, size_t ws_bytes, float* scores, float* lat_v, float* lat_g,
                      float* pred_v, float* pred_g, int32_t* err, void* stream) {
  if (!m || !ws || !err) return FS_EINVAL;
  if (!fs_model_supports(m, precision)) return FS_ENOTSUP;
  const int P = n_poses;
  if (P <= 0) return FS_OK;
  const bool want_v = heads & 1, want_g = heads & 2, want_f = heads & 4;
  const fs_model_desc& d = m->d;
  const bool late = d.fusion_mode == FS_MODE_LATE;
  const bool need_v = want_v || want_f, need_g = want_g || want_f;
  if (need_v && !grids) return FS_EINVAL;
  if (need_g && (!feats || !node_off)) return FS_EINVAL;
  if (want_f && !scores) return FS_EINVAL;
  const int64_t E = 2 * (n_cov > n_ncov ? n_cov : n_ncov);
  // per-pose node bound: the caller's (checked on device), else the worst case
  const int64_t bound = max_pose_nodes > 0 ? (max_pose_nodes < n_nodes ? max_pose_nodes : n_nodes)
                                           : (n_nodes < FS_MAX_POSE_ATOMS ? n_nodes : FS_MAX_POSE_ATOMS);
  WsPlan w = plan_ws(*m, P, n_nodes, E, precision, bound);
  char* W = (char*)(((uintptr_t)ws + 255) & ~(uintptr_t)255);
  if ((size_t)(W - (char*)ws) + w.total > ws_bytes) return FS_ECAPACITY;
  cudaStream_t st = (cudaStream_t)stream;
  int rc;
  FS_CUDA_CHECK(cudaMemsetAsync(err, 0, 4 * (size_t)P, st));
  if (need_v) {
    if (precision == FS_PREC_MIXED) {
      if ((rc = launch_grid_convert(grids, W + w.grid, P, m->cin, m->G, false, err, st))) return rc;
      if ((rc = launch_split_bf16((const float*)(W + w.grid), (__nv_bfloat16*)(W + w.grid_hi),
                                  (__nv_bfloat16*)(W + w.grid_lo), (int64_t)P * m->G * m->G * m->G * m->cin, st)))
        return rc;
      if ((rc = umma::voxel_convs_x3(d, (const char*)m->blob + m->umma_off, m->P(m->c1b), m->P(m->c2b),
                                     m->P(m->c3b), m->P(m->c4b), P, (const __nv_bfloat16*)(W + w.grid_hi),
                                     (const __nv_bfloat16*)(W + w.grid_lo), W + w.umma, (float*)(W + w.p2), st)))
        return rc;
    } else if (precision != FS_PREC_FP32) {
      if ((rc = launch_grid_convert(grids, W + w.grid, P, m->cin, m->G, true, err, st))) return rc;
      if ((rc = umma::voxel_convs(d, (const char*)m->blob + m->umma_off, m->P(m->c1b), m->P(m->c2b),
                                  m->P(m->c3b), m->P(m->c4b), P, (const __nv_bfloat16*)(W + w.grid),
                                  W + w.umma, (float*)(W + w.p2), st)))
        return rc;
    } else {
      if ((rc = launch_grid_convert(grids, W + w.grid, P, m->cin, m->G, false, err, st))) return rc;
      if ((rc = voxel_head_fp32(*m, P, W, w, st))) return rc;
    }
    if ((rc = voxel_tail(*m, P, W, w, late || pred_v, st, precision == FS_PREC_BF16))) return rc;
  }
  if (need_g) {
    int64_t* noff = (int64_t*)(W + w.node_off);
    FS_CUDA_CHECK(cudaMemcpyAsync(noff, node_off, 8 * (size_t)(P + 1), cudaMemcpyDeviceToDevice, st));
    int32_t* node_pose = (int32_t*)(W + w.node_pose);
    int64_t* cursor = (int64_t*)(W + w.cursor);
    const size_t scan_b = scan_ws_bytes(n_nodes > P ? n_nodes : P) + 1024;
    if ((rc = launch_csr_from_edges(cov_edges, n_cov, noff, P, n_nodes, node_pose, (int32_t*)(W + w.deg_cov),
                                    (int64_t*)(W + w.row_cov), cursor, (col_t*)(W + w.col_cov), W + w.scan, scan_b,
                                    st)))
      return rc;
    if ((rc = launch_csr_from_edges(ncov_edges, n_ncov, noff, P, n_nodes, node_pose, (int32_t*)(W + w.deg_ncov),
                                    (int64_t*)(W + w.row_ncov), cursor, (col_t*)(W + w.col_ncov), W + w.scan,
                                    scan_b, st)))
      return rc;
    if ((rc = launch_f64_to_f32(feats, (float*)(W + w.feats), n_nodes * m->F, m->F, node_pose, err, st))) return rc;
    // the per-pose node bound sizes the SG-CNN's shared-memory node state (and
    // picks the tensor-core kernel when it fits); poses above it are flagged
    if ((rc = launch_pose_bound(noff, P, bound, err, st))) return rc;
    if ((rc = graph_head(*m, P, (int)(bound < FS_MAX_POSE_ATOMS ? bound : FS_MAX_POSE_ATOMS), W, w, err,
                         late || pred_g, precision, st, nullptr, false)))
      return rc;
  }
  if (want_f) {
    if (!late && (rc = fusion_head(*m, P, W, w, scores, st))) return rc;
    if ((rc = launch_finalize(P, d.fusion_mode, (float*)(W + w.pv), (float*)(W + w.pg), scores, err, st))) return rc;
  }
  return copy_outputs(*m, P, W, w, want_v || want_f ? lat_v : nullptr, want_g || want_f ? lat_g : nullptr,
                      pred_v, pred_g, st);
}

int fs_debug_conv(const fs_model* m, int layer, int32_t n_poses, const void* in, const void* residual, void* out,
                  void* stream) {
  if (!m || !in || !out || n_poses < 0) return FS_EINVAL;
  if (!m->umma_ok) return FS_ENOTSUP;
  const float* bias[5] = {nullptr, m->P(m->c1b), m->P(m->c2b), m->P(m->c3b), m->P(m->c4b)};
  if (layer < 1 || layer > 4) return FS_EINVAL;
  return umma::debug_layer(m->d, (const char*)m->blob + m->umma_off, bias[layer], nullptr, layer, n_poses, in,
                           residual, out, (cudaStream_t)stream);
}

// ---- inspection of the scoring-path radius graph ---------------------------
struct GraphHookPlan {
  size_t total = 0, node_off, scan, row_c, row_n, deg_c, deg_n, col_c, col_n, feats, cnt, aff;
  int64_t N, S;
  size_t take(size_t bytes) { size_t o = total; total = align_up(total + bytes, 256); return o; }
};

static GraphHookPlan graph_hook_plan(int64_t P, int max_atoms, int64_t max_edges, int factored, int c_elem) {
  GraphHookPlan g;
  g.S = factored ? fact_slice_rows(max_atoms) : max_atoms;
  g.N = P * g.S;
  g.node_off = g.take(8 * (P + 1));
  g.scan = g.take(scan_ws_bytes(g.N > P ? g.N : P) + 1024);
  g.row_c = g.take(8 * (g.N + 1)); g.row_n = g.take(8 * (g.N + 1));
  g.deg_c = g.take(4 * g.N); g.deg_n = g.take(4 * g.N);
  g.col_c = g.take(sizeof(col_t) * P * max_edges); g.col_n = g.take(sizeof(col_t) * P * max_edges);
  g.feats = g.take(4 * g.N * (c_elem + 4));
  g.cnt = g.take(8 * P); g.aff = g.take(4 * g.N);
  return g;
}

size_t fs_scoring_graph_ws_bytes(int32_t n_poses, int32_t max_pose_atoms, int64_t max_edges, int32_t factored,
                                 int32_t c_elem) {
  if (n_poses < 0 || max_edges <= 0 || c_elem < 1) return 0;
  const int max_atoms = max_pose_atoms > 0 ? max_pose_atoms : FS_MAX_POSE_ATOMS;
  return graph_hook_plan(n_poses, max_atoms, max_edges, factored, c_elem).total + 256;
}

int fs_scoring_graph(const fs_pose_batch* b, double cov_thresh, double noncov_thresh, int64_t max_edges,
                     int32_t factored, int32_t max_pocket_atoms, int32_t c_elem, double box_size, void* ws,
                     size_t ws_bytes, int32_t* n_cov, int32_t* n_ncov, int32_t* ent_cov, int32_t* ent_ncov,
                     double* d_cov, double* d_ncov, int32_t* err, void* stream) {
  if (!b || !ws || !n_cov || !n_ncov || !ent_cov || !ent_ncov || !err || max_edges <= 0 || c_elem < 1)
    return FS_EINVAL;
  const int P = b->n_poses;
  if (P <= 0) return FS_OK;
  const int max_atoms = b->max_pose_atoms > 0 ? b->max_pose_atoms : FS_MAX_POSE_ATOMS;
  const GraphHookPlan g = graph_hook_plan(P, max_atoms, max_edges, factored, c_elem);
  char* W = (char*)(((uintptr_t)ws + 255) & ~(uintptr_t)255);
  if ((size_t)(W - (char*)ws) + g.total > ws_bytes) return FS_ECAPACITY;
  cudaStream_t st = (cudaStream_t)stream;
  int rc;
  FS_CUDA_CHECK(cudaMemsetAsync(err, 0, 4 * (size_t)P, st));
  int64_t* node_off = (int64_t*)(W + g.node_off);
  int32_t* cnt = nullptr; int32_t* aff = nullptr;
  if (factored) {
    // exactly fs_score_poses_cached's graph launch
    if (max_pocket_atoms <= 0 || max_pocket_atoms > FS_MAX_POSE_ATOMS) return FS_EINVAL;
    cnt = (int32_t*)(W + g.cnt); aff = (int32_t*)(W + g.aff);
    if ((rc = launch_graph_fact(*b, cov_thresh, noncov_thresh, box_size, c_elem, g.S, max_edges, max_pocket_atoms,
                                cnt, aff, (float*)(W + g.feats), (int64_t*)(W + g.row_c), (int32_t*)(W + g.deg_c),
                                (col_t*)(W + g.col_c), (int64_t*)(W + g.row_n), (int32_t*)(W + g.deg_n),
                                (col_t*)(W + g.col_n), err, st)))
      return rc;
  } else {
    // exactly fs_score_poses's node offsets + graph launch
    if ((rc = launch_node_offsets(*b, node_off, W + g.scan, scan_ws_bytes(g.N > P ? g.N : P) + 1024, st,
                                  max_atoms)))
      return rc;
    if ((rc = launch_graph_csr(*b, node_off, cov_thresh, noncov_thresh, (int64_t*)(W + g.row_c),
                               (int32_t*)(W + g.deg_c), (col_t*)(W + g.col_c), nullptr, (int64_t*)(W + g.row_n),
                               (int32_t*)(W + g.deg_n), (col_t*)(W + g.col_n), nullptr, max_edges, err, st,
                               (float*)(W + g.feats), c_elem, box_size)))
      return rc;
  }
  return launch_csr_entries(*b, node_off, cnt, aff, g.S, max_edges, (int)g.S, (int64_t*)(W + g.row_c),
                            (int32_t*)(W + g.deg_c), (col_t*)(W + g.col_c), (int64_t*)(W + g.row_n),
                            (int32_t*)(W + g.deg_n), (col_t*)(W + g.col_n), max_edges, n_cov, n_ncov, ent_cov,
                            ent_ncov, d_cov, d_ncov, err, st);
}

size_t fs_topk_ws_bytes(int64_t n) { return topk_ws_bytes(n); }

int fs_topk_merge(const float* a_scores, const int64_t* a_idx, int64_t na, const float* b_scores,
                  const int64_t* b_idx, int64_t nb, int32_t k, float* out_scores, int64_t* out_idx, void* ws,
                  size_t ws_bytes, void* stream) {
  if (na < 0 || nb < 0 || !out_scores || !out_idx) return FS_EINVAL;
  return launch_topk_merge(a_scores, a_idx, na, b_scores, b_idx, nb, k, out_scores, out_idx, ws, ws_bytes,
                           (cudaStream_t)stream);
}

int fs_best_pose(const int64_t* compound, const int64_t* pose_id, const float* scores, int64_t n,
                 int64_t n_compounds, int32_t direction, int64_t* best_idx, uint64_t* best_key, void* stream) {
  if (!compound || !pose_id || !scores || !best_idx || !best_key || n < 0) return FS_EINVAL;
  return launch_best_pose(compound, pose_id, scores, n, n_compounds, direction, best_idx, best_key,
                          (cudaStream_t)stream);
}

int fs_best_pose_update(const int64_t* compound, int64_t compound_base, const int64_t* pose_id, const float* scores,
                        int64_t n, int64_t n_compounds, int32_t direction, uint64_t* best_key, void* stream) {
  if (!compound || !pose_id || !scores || !best_key || n < 0 || n_compounds < 0) return FS_EINVAL;
  return launch_best_update(compound, compound_base, pose_id, scores, n, n_compounds, direction, best_key,
                            (cudaStream_t)stream);
}

int fs_best_pose_decode(const uint64_t* best_key, int64_t n_compounds, int32_t direction, float* best_score,
                        int64_t* best_pose, void* stream) {
  if (!best_key || !best_score || !best_pose || n_compounds < 0) return FS_EINVAL;
  return launch_best_decode(best_key, n_compounds, direction, best_score, best_pose, (cudaStream_t)stream);
}

}  // extern "C"
