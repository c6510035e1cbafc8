// Featurizer kernels: voxel splat and exact radius graph (sm_100a).
//
// Reference: complexes.py:171-184 (voxelize), :223-254 (build_graph),
// models.py:233-256 (batch_graphs -> symmetric CSR adjacency).
#include <cub/cub.cuh>

#include "common.cuh"

namespace fs {

// ---------------------------------------------------------------------------
// node offsets
// ---------------------------------------------------------------------------
// clamp > 0: a pose above `clamp` nodes (flagged FS_ERR_TOO_LARGE by the graph
// kernels) occupies only `clamp` node rows, so one oversize pose can neither
// push the others past a workspace sized P * clamp nor be written past it
__global__ void pose_node_counts_kernel(fs_pose_batch b, int64_t* counts, int64_t clamp) {
  int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= b.n_poses) return;
  int t = b.pose_target ? b.pose_target[p] : -1;
  int64_t n = b.atom_off[p + 1] - b.atom_off[p];
  if (t >= 0) n += b.pocket_off[t + 1] - b.pocket_off[t];
  counts[p] = clamp > 0 && n > clamp ? clamp : n;
}

// ---------------------------------------------------------------------------
// voxelize: one CTA per pose.  idx = clip(floor(((pos + box/2)/box)*G), 0, G-1)
// in float64 with the reference's operation order (complexes.py:180-181);
// channel = role*c_elem + clip(elem, 0, c_elem-1) (:182); +1.0 per atom (:183).
// Counts are integers, so the accumulation order is irrelevant (exact).
// Fast path: splat into a shared-memory u32 grid, then one coalesced store.
// ---------------------------------------------------------------------------
struct VoxParams {
  int g, c_elem, channels, layout;
  double half, box, gd;
};

__device__ __forceinline__ int vox_axis(double x, const VoxParams& v, bool& nan) {
  double t = __dmul_rn(__ddiv_rn(__dadd_rn(x, v.half), v.box), v.gd);
  if (isnan(t)) { nan = true; return 0; }
  t = floor(t);
  t = fmin(fmax(t, 0.0), (double)(v.g - 1));   // np.clip on the float index
  return (int)t;
}

__device__ __forceinline__ int64_t vox_index(int ch, int ix, int iy, int iz, const VoxParams& v) {
  const int64_t g = v.g;
  if (v.layout == FS_GRID_NCDHW_F64) return ((ch * g + ix) * g + iy) * g + iz;
  return (((int64_t)ix * g + iy) * g + iz) * v.channels + ch;     // NDHWC
}

__global__ void voxelize_smem_kernel(fs_pose_batch b, VoxParams v, void* out, int32_t* err) {
  extern __shared__ uint32_t cnt[];
  const int p = blockIdx.x;
  const int64_t cells = (int64_t)v.channels * v.g * v.g * v.g;
  for (int64_t i = threadIdx.x; i < cells; i += blockDim.x) cnt[i] = 0u;
  __syncthreads();
  PoseView pv = pose_view(b, p);
  int flags = 0;
  for (int64_t i = threadIdx.x; i < pv.n(); i += blockDim.x) {
    double x, y, z; int32_t e, r;
    pv.atom(i, x, y, z, e, r);
    if (r != 0 && r != 1) { flags |= FS_ERR_ROLE; continue; }
    bool nan = false;
    int ix = vox_axis(x, v, nan), iy = vox_axis(y, v, nan), iz = vox_axis(z, v, nan);
    if (nan) { flags |= FS_ERR_NAN; continue; }
    int ch = r * v.c_elem + min(max(e, 0), v.c_elem - 1);
    atomicAdd(&cnt[vox_index(ch, ix, iy, iz, v)], 1u);
  }
  if (flags) atomicOr(&err[p], flags);
  __syncthreads();
  if (v.layout == FS_GRID_NCDHW_F64) {
    double* o = (double*)out + (int64_t)p * cells;
    for (int64_t i = threadIdx.x; i < cells; i += blockDim.x) o[i] = (double)cnt[i];
  } else if (v.layout == FS_GRID_NDHWC_F32) {
    float* o = (float*)out + (int64_t)p * cells;
    for (int64_t i = threadIdx.x; i < cells; i += blockDim.x) o[i] = (float)cnt[i];
  } else {
    __nv_bfloat16* o = (__nv_bfloat16*)out + (int64_t)p * cells;
    for (int64_t i = threadIdx.x; i < cells; i += blockDim.x) o[i] = __float2bfloat16_rn((float)cnt[i]);
  }
}

// bf16 NDHWC with a multiple of 8 channels (the tcgen05 conv input): counts
// packed two per 32-bit shared word (a count never exceeds the pose's atom
// count, < 2^16, so a half never carries into the other), half the shared
// memory of the u32 grid (3 CTAs per SM instead of 1); one 16-byte store per
// 8 channels of a voxel.  Same values as voxelize_smem_kernel (counts are
// exact in fp32, one RN rounding to bf16).
__global__ void voxelize_bf16_kernel(fs_pose_batch b, VoxParams v, __nv_bfloat16* out, int32_t* err) {
  extern __shared__ uint4 cnt4[];
  uint32_t* cnt = reinterpret_cast<uint32_t*>(cnt4);
  const int p = blockIdx.x;
  const int vox = v.g * v.g * v.g, wpv = v.channels / 2;   // words per voxel
  const int words = vox * wpv;
  for (int i = threadIdx.x; i < words / 4; i += blockDim.x) cnt4[i] = make_uint4(0u, 0u, 0u, 0u);
  __syncthreads();
  PoseView pv = pose_view(b, p);
  int flags = 0;
  for (int64_t i = threadIdx.x; i < pv.n(); i += blockDim.x) {
    double x, y, z; int32_t e, r;
    pv.atom(i, x, y, z, e, r);
    if (r != 0 && r != 1) { flags |= FS_ERR_ROLE; continue; }
    bool nan = false;
    int ix = vox_axis(x, v, nan), iy = vox_axis(y, v, nan), iz = vox_axis(z, v, nan);
    if (nan) { flags |= FS_ERR_NAN; continue; }
    const int ch = r * v.c_elem + min(max(e, 0), v.c_elem - 1);
    const int vi = (ix * v.g + iy) * v.g + iz;
    atomicAdd(&cnt[vi * wpv + (ch >> 1)], (ch & 1) ? 65536u : 1u);
  }
  if (flags) atomicOr(&err[p], flags);
  __syncthreads();
  uint4* o = reinterpret_cast<uint4*>(out + (int64_t)p * vox * v.channels);
  for (int i = threadIdx.x; i < words / 4; i += blockDim.x) {   // 8 channels per 16-byte store
    const uint4 c = cnt4[i];
    uint4 pk;
    __nv_bfloat162* b2 = reinterpret_cast<__nv_bfloat162*>(&pk);
    b2[0] = __floats2bfloat162_rn((float)(c.x & 0xffffu), (float)(c.x >> 16));
    b2[1] = __floats2bfloat162_rn((float)(c.y & 0xffffu), (float)(c.y >> 16));
    b2[2] = __floats2bfloat162_rn((float)(c.z & 0xffffu), (float)(c.z >> 16));
    b2[3] = __floats2bfloat162_rn((float)(c.w & 0xffffu), (float)(c.w >> 16));
    o[i] = pk;
  }
}

// Large grids: global atomics into a zeroed output (fp64 / fp32 layouts only).
__global__ void voxelize_global_kernel(fs_pose_batch b, VoxParams v, void* out, int32_t* err) {
  const int p = blockIdx.x;
  const int64_t cells = (int64_t)v.channels * v.g * v.g * v.g;
  PoseView pv = pose_view(b, p);
  int flags = 0;
  for (int64_t i = threadIdx.x; i < pv.n(); i += blockDim.x) {
    double x, y, z; int32_t e, r;
    pv.atom(i, x, y, z, e, r);
    if (r != 0 && r != 1) { flags |= FS_ERR_ROLE; continue; }
    bool nan = false;
    int ix = vox_axis(x, v, nan), iy = vox_axis(y, v, nan), iz = vox_axis(z, v, nan);
    if (nan) { flags |= FS_ERR_NAN; continue; }
    int ch = r * v.c_elem + min(max(e, 0), v.c_elem - 1);
    int64_t idx = (int64_t)p * cells + vox_index(ch, ix, iy, iz, v);
    if (v.layout == FS_GRID_NCDHW_F64) atomicAdd((double*)out + idx, 1.0);
    else atomicAdd((float*)out + idx, 1.0f);
  }
  if (flags) atomicOr(&err[p], flags);
}

// ---------------------------------------------------------------------------
// node features [onehot(clip elem) | role | pos/box + 0.5] (complexes.py:233-236)
// ---------------------------------------------------------------------------
template <typename T>
__global__ void node_features_kernel(fs_pose_batch b, const int64_t* node_off, int c_elem,
                                     double box, T* out) {
  const int p = blockIdx.x;
  PoseView pv = pose_view(b, p);
  const int F = c_elem + 4;
  T* o = out + node_off[p] * F;
  for (int64_t i = threadIdx.x; i < pv.n(); i += blockDim.x) {
    double x, y, z; int32_t e, r;
    pv.atom(i, x, y, z, e, r);
    T* f = o + i * F;
    int ec = min(max(e, 0), c_elem - 1);
    for (int c = 0; c < c_elem; ++c) f[c] = (T)(c == ec ? 1.0 : 0.0);
    f[c_elem] = (T)r;
    f[c_elem + 1] = (T)__dadd_rn(__ddiv_rn(x, box), 0.5);
    f[c_elem + 2] = (T)__dadd_rn(__ddiv_rn(y, box), 0.5);
    f[c_elem + 3] = (T)__dadd_rn(__ddiv_rn(z, box), 0.5);
  }
}

// ---------------------------------------------------------------------------
// Radius graph.  One CTA per pose, two passes (count, fill) sharing code.
//   covalent     : same role,  d <= t_cov   -- cell list, cells >= t_cov wide
//   non-covalent : other role, d <= t_ncov  -- scan of the other role's atoms
// Exact predicate (float64, no FMA): d2 = (dx*dx+dy*dy)+dz*dz; candidate iff
// d2 <= rmax*rmax (cKDTree.query_pairs, complexes.py:237-238); keep iff
// sqrt(d2) <= t (np.linalg.norm, :241-244).  A float32 prefilter with a
// 1e-3 A margin only skips pairs that are certainly too far.
// Rows are written by one thread each (deterministic); covalent rows are then
// insertion-sorted so every row is ascending in the neighbour id.
// ---------------------------------------------------------------------------
constexpr int kGraphThreads = 256;
constexpr int kMaxCellsAxis = 12;

struct GraphSmem {
  float4* pf;        // x, y, z (fp32), role (as float)       [n]
  int* cell_list;    // atom ids sorted by (role, cell)       [n]
  int* role_list;    // atom ids sorted by (role, id)         [n]
  int* keys;         // (role, cell) key per atom             [n]
  int* cell_start;   // [2*NC + 1]
};

__host__ __device__ inline size_t graph_smem_bytes(int n) {
  return (size_t)n * (16 + 4 + 4 + 4) + (size_t)(2 * kMaxCellsAxis * kMaxCellsAxis * kMaxCellsAxis + 2) * 4 + 64;
}

__device__ __forceinline__ double block_reduce_minmax(double v, bool is_max, double* scratch) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int o = 16; o > 0; o >>= 1) {
    double w = __shfl_xor_sync(0xffffffffu, v, o);
    v = is_max ? fmax(v, w) : fmin(v, w);
  }
  __syncthreads();
  if (lane == 0) scratch[warp] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    double r = scratch[0];
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) r = is_max ? fmax(r, scratch[w]) : fmin(r, scratch[w]);
    scratch[32] = r;
  }
  __syncthreads();
  return scratch[32];
}

template <bool FILL>
__global__ void __launch_bounds__(kGraphThreads)
graph_kernel(fs_pose_batch b, const int64_t* __restrict__ node_off, double tc, double tn,
             int32_t* deg_cov, int32_t* deg_ncov,
             const int64_t* __restrict__ row_cov, const int64_t* __restrict__ row_ncov,
             int32_t* col_cov, int32_t* col_ncov, double* dist_cov, double* dist_ncov,
             int64_t cap_cov, int64_t cap_ncov, int32_t* err, int smem_atoms) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ double red[33];
  __shared__ int s_flags, s_role_cnt[2];
  __shared__ double s_min[3];

  const int p = blockIdx.x;
  PoseView pv = pose_view(b, p);
  const int n = (int)pv.n();
  const int64_t base = node_off[p];
  if (threadIdx.x == 0) { s_flags = 0; s_role_cnt[0] = 0; s_role_cnt[1] = 0; }
  if (n > smem_atoms) {
    if (threadIdx.x == 0) atomicOr(&err[p], FS_ERR_TOO_LARGE);
    if (!FILL) for (int i = threadIdx.x; i < n; i += blockDim.x) { deg_cov[base + i] = 0; deg_ncov[base + i] = 0; }
    return;
  }
  GraphSmem s;
  s.pf = (float4*)smem_raw;
  s.cell_list = (int*)(s.pf + smem_atoms);
  s.role_list = s.cell_list + smem_atoms;
  s.keys = s.role_list + smem_atoms;
  s.cell_start = s.keys + smem_atoms;
  __syncthreads();

  // ---- load atoms, validate, bounding box --------------------------------
  double lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
  int flags = 0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    double x, y, z; int32_t e, r;
    pv.atom(i, x, y, z, e, r);
    if (r != 0 && r != 1) flags |= FS_ERR_ROLE;
    if (!isfinite(x) || !isfinite(y) || !isfinite(z)) flags |= FS_ERR_NONFINITE;
    s.pf[i] = make_float4((float)x, (float)y, (float)z, (float)r);
    lo[0] = fmin(lo[0], x); lo[1] = fmin(lo[1], y); lo[2] = fmin(lo[2], z);
    hi[0] = fmax(hi[0], x); hi[1] = fmax(hi[1], y); hi[2] = fmax(hi[2], z);
  }
  if (flags) atomicOr(&s_flags, flags);
  double ext_max = 0.0, absmax = 0.0;
  for (int a = 0; a < 3; ++a) {
    double l = block_reduce_minmax(lo[a], false, red);
    double h = block_reduce_minmax(hi[a], true, red);
    if (threadIdx.x == 0) s_min[a] = l;
    ext_max = fmax(ext_max, h - l);
    absmax = fmax(absmax, fmax(fabs(l), fabs(h)));
  }
  __syncthreads();
  if (s_flags) {
    if (threadIdx.x == 0) atomicOr(&err[p], s_flags);
    if (!FILL) for (int i = threadIdx.x; i < n; i += blockDim.x) { deg_cov[base + i] = 0; deg_ncov[base + i] = 0; }
    return;
  }
  const bool prefilter = absmax < 1024.0;   // fp32 coordinate error <= 6.1e-5 A
  // cell edge >= t_cov so covalent partners sit in adjacent cells; ext_max
  // bounds every axis, so one count per axis suffices.
  const double cs = fmax(tc * 1.0001, ext_max / (kMaxCellsAxis - 1));
  const int nc_axis = min(kMaxCellsAxis, (int)floor(ext_max / cs) + 1);
  const int NC = nc_axis * nc_axis * nc_axis;
  for (int i = threadIdx.x; i < 2 * NC + 2; i += blockDim.x) s.cell_start[i] = 0;
  __syncthreads();

  auto cell_coord = [&](double x, int a) -> int {
    int c = (int)floor(__ddiv_rn(__dsub_rn(x, s_min[a]), cs));
    return min(max(c, 0), nc_axis - 1);
  };
  // ---- counting sort by (role, cell) --------------------------------------
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    double x, y, z; int32_t e, r;
    pv.atom(i, x, y, z, e, r);
    int c = (cell_coord(x, 0) * nc_axis + cell_coord(y, 1)) * nc_axis + cell_coord(z, 2);
    s.keys[i] = r * NC + c;
    atomicAdd(&s.cell_start[r * NC + c + 1], 1);
    atomicAdd(&s_role_cnt[r], 1);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int k = 1; k <= 2 * NC; ++k) s.cell_start[k] += s.cell_start[k - 1];
  }
  __syncthreads();
  // role_list: stable partition by role, ascending id (ballot scan per tile)
  {
    __shared__ int warp_cnt[2][kGraphThreads / 32];
    __shared__ int run[2];
    if (threadIdx.x == 0) { run[0] = 0; run[1] = s_role_cnt[0]; }
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int t0 = 0; t0 < n; t0 += blockDim.x) {
      int i = t0 + threadIdx.x;
      int r = (i < n) ? (int)s.pf[i].w : -1;
      unsigned m0 = __ballot_sync(0xffffffffu, r == 0), m1 = __ballot_sync(0xffffffffu, r == 1);
      if (lane == 0) { warp_cnt[0][warp] = __popc(m0); warp_cnt[1][warp] = __popc(m1); }
      __syncthreads();
      if (r >= 0) {
        unsigned m = r == 0 ? m0 : m1;
        int pos = run[r] + __popc(m & ((1u << lane) - 1u));
        for (int w = 0; w < warp; ++w) pos += warp_cnt[r][w];
        s.role_list[pos] = i;
      }
      __syncthreads();
      if (threadIdx.x == 0) {
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) { run[0] += warp_cnt[0][w]; run[1] += warp_cnt[1][w]; }
      }
      __syncthreads();
    }
  }
  // scatter atoms into cell order (order within a cell is irrelevant: covalent
  // rows are sorted afterwards).  cell_start acts as a cursor, then shifts back.
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    int slot = atomicAdd(&s.cell_start[s.keys[i]], 1);
    s.cell_list[slot] = i;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int k = 2 * NC; k > 0; --k) s.cell_start[k] = s.cell_start[k - 1];
    s.cell_start[0] = 0;
  }
  __syncthreads();

  const int nrole0 = s_role_cnt[0];
  const float tcf = (float)tc + 1e-3f, tnf = (float)tn + 1e-3f;
  const float tcf2 = tcf * tcf, tnf2 = tnf * tnf;
  const double rmax = fmax(tc, tn);
  const double rmax2 = __dmul_rn(rmax, rmax);

  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    double xi, yi, zi; int32_t ei, ri;
    pv.atom(i, xi, yi, zi, ei, ri);
    const float4 fi = s.pf[i];
    const int cx = cell_coord(xi, 0), cy = cell_coord(yi, 1), cz = cell_coord(zi, 2);
    // ---- covalent row ----
    int64_t wc = FILL ? row_cov[base + i] : 0;
    const int64_t ec = FILL ? row_cov[base + i + 1] : 0;
    int cnt_c = 0;
    for (int dx = -1; dx <= 1; ++dx) {
      int ax = cx + dx; if (ax < 0 || ax >= nc_axis) continue;
      for (int dy = -1; dy <= 1; ++dy) {
        int ay = cy + dy; if (ay < 0 || ay >= nc_axis) continue;
        for (int dz = -1; dz <= 1; ++dz) {
          int az = cz + dz; if (az < 0 || az >= nc_axis) continue;
          int key = ri * NC + (ax * nc_axis + ay) * nc_axis + az;
          for (int q = s.cell_start[key]; q < s.cell_start[key + 1]; ++q) {
            int j = s.cell_list[q];
            if (j == i) continue;
            float4 fj = s.pf[j];
            if (prefilter) {
              float ddx = fi.x - fj.x, ddy = fi.y - fj.y, ddz = fi.z - fj.z;
              if (ddx * ddx + ddy * ddy + ddz * ddz > tcf2) continue;
            }
            double xj, yj, zj; int32_t ej, rj;
            pv.atom(j, xj, yj, zj, ej, rj);
            double d2 = dist2_exact(xi - xj, yi - yj, zi - zj);
            if (!(d2 <= rmax2)) continue;
            double d = __dsqrt_rn(d2);
            if (!(d <= tc)) continue;
            if (FILL) {
              if (wc < ec && ec <= cap_cov) {
                col_cov[wc] = j;
                if (dist_cov) dist_cov[wc] = d;
              }
              ++wc;
            } else {
              ++cnt_c;
            }
          }
        }
      }
    }
    // ---- non-covalent row: other role, ascending id ----
    const int o_begin = ri == 0 ? nrole0 : 0, o_end = ri == 0 ? n : nrole0;
    int64_t wn = FILL ? row_ncov[base + i] : 0;
    const int64_t en = FILL ? row_ncov[base + i + 1] : 0;
    int cnt_n = 0;
    for (int q = o_begin; q < o_end; ++q) {
      int j = s.role_list[q];
      float4 fj = s.pf[j];
      if (prefilter) {
        float ddx = fi.x - fj.x, ddy = fi.y - fj.y, ddz = fi.z - fj.z;
        if (ddx * ddx + ddy * ddy + ddz * ddz > tnf2) continue;
      }
      double xj, yj, zj; int32_t ej, rj;
      pv.atom(j, xj, yj, zj, ej, rj);
      double d2 = dist2_exact(xi - xj, yi - yj, zi - zj);
      if (!(d2 <= rmax2)) continue;
      double d = __dsqrt_rn(d2);
      if (!(d <= tn)) continue;
      if (FILL) {
        if (wn < en && en <= cap_ncov) {
          col_ncov[wn] = j;
          if (dist_ncov) dist_ncov[wn] = d;
        }
        ++wn;
      } else {
        ++cnt_n;
      }
    }
    if (!FILL) {
      deg_cov[base + i] = cnt_c;
      deg_ncov[base + i] = cnt_n;
    } else {
      if (ec > cap_cov || en > cap_ncov) {
        atomicOr(&err[p], FS_ERR_EDGE_CAP);
      } else {
        // insertion sort of the covalent row (short; cell order -> id order)
        const int64_t rb = row_cov[base + i];
        for (int64_t a = rb + 1; a < ec; ++a) {
          int v = col_cov[a];
          double dv = dist_cov ? dist_cov[a] : 0.0;
          int64_t c = a - 1;
          while (c >= rb && col_cov[c] > v) {
            col_cov[c + 1] = col_cov[c];
            if (dist_cov) dist_cov[c + 1] = dist_cov[c];
            --c;
          }
          col_cov[c + 1] = v;
          if (dist_cov) dist_cov[c + 1] = dv;
        }
      }
    }
  }
}

// ---------------------------------------------------------------------------
// CSR helpers
// ---------------------------------------------------------------------------
__global__ void widen_kernel(const int32_t* deg, int64_t n, int64_t* out) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = deg[i];
  if (i == n) out[n] = 0;
}

// per-row count of entries with col > row (pose-local ids)
__global__ void upper_counts_kernel(const int64_t* node_off, int n_poses, const int64_t* row_ptr,
                                    const int32_t* col, int64_t* pose_cnt) {
  const int p = blockIdx.x;
  const int64_t base = node_off[p], n = node_off[p + 1] - base;
  int64_t c = 0;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x)
    for (int64_t q = row_ptr[base + i]; q < row_ptr[base + i + 1]; ++q) c += (col[q] > i);
  typedef cub::BlockReduce<int64_t, 256> BR;
  __shared__ typename BR::TempStorage tmp;
  int64_t tot = BR(tmp).Sum(c);
  if (threadIdx.x == 0) pose_cnt[p] = tot;
}

// one warp per pose row sweep keeps lexicographic (i, j) order: rows in
// ascending i, each row ascending j.
__global__ void upper_edges_kernel(const int64_t* node_off, int n_poses, const int64_t* row_ptr,
                                   const int32_t* col, const double* dist, const int64_t* edge_off,
                                   int64_t* edges, double* dists) {
  const int p = blockIdx.x;
  if (threadIdx.x >= 32) return;
  const int lane = threadIdx.x;
  const int64_t base = node_off[p], n = node_off[p + 1] - base;
  int64_t w = edge_off[p];
  for (int64_t i = 0; i < n; ++i) {
    const int64_t rb = row_ptr[base + i], re = row_ptr[base + i + 1];
    for (int64_t q0 = rb; q0 < re; q0 += 32) {
      int64_t q = q0 + lane;
      bool take = q < re && col[q] > i;
      unsigned m = __ballot_sync(0xffffffffu, take);
      if (take) {
        int64_t o = w + __popc(m & ((1u << lane) - 1u));
        edges[2 * o] = i;
        edges[2 * o + 1] = col[q];
        if (dists) dists[o] = dist[q];
      }
      w += __popc(m);
    }
  }
}

// CSR from i<j edge lists with GLOBAL node ids (pre-featurized batch path,
// models.py:238-247 builds the same symmetric 0/1 matrix).
__global__ void node_pose_kernel(const int64_t* node_off, int n_poses, int32_t* node_pose) {
  const int p = blockIdx.x;
  for (int64_t i = node_off[p] + threadIdx.x; i < node_off[p + 1]; i += blockDim.x) node_pose[i] = p;
}

__global__ void edge_degree_kernel(const int64_t* edges, int64_t ne, int32_t* deg) {
  int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= ne) return;
  atomicAdd(&deg[edges[2 * e]], 1);
  atomicAdd(&deg[edges[2 * e + 1]], 1);
}

__global__ void edge_fill_kernel(const int64_t* edges, int64_t ne, const int64_t* node_off,
                                 const int32_t* node_pose, int64_t* cursor, col_t* col) {
  int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= ne) return;
  int64_t i = edges[2 * e], j = edges[2 * e + 1];
  int64_t oi = node_off[node_pose[i]], oj = node_off[node_pose[j]];
  unsigned long long si = atomicAdd((unsigned long long*)&cursor[i], 1ull);
  unsigned long long sj = atomicAdd((unsigned long long*)&cursor[j], 1ull);
  col[si] = (col_t)(j - oj);
  col[sj] = (col_t)(i - oi);
}

__global__ void sort_rows_kernel(const int64_t* row_ptr, int64_t n, col_t* col) {
  int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n) return;
  const int64_t rb = row_ptr[r], re = row_ptr[r + 1];
  for (int64_t a = rb + 1; a < re; ++a) {
    int v = col[a];
    int64_t c = a - 1;
    while (c >= rb && col[c] > v) { col[c + 1] = col[c]; --c; }
    col[c + 1] = v;
  }
}

// ---------------------------------------------------------------------------
// host launchers (used by abi.cu)
// ---------------------------------------------------------------------------
size_t scan_ws_bytes(int64_t n) {
  size_t bytes = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, bytes, (int64_t*)nullptr, (int64_t*)nullptr, (int)(n + 1));
  return bytes + 256;
}

int exclusive_scan_i64(int64_t* inout, int64_t n_plus_1, void* ws, size_t ws_bytes, cudaStream_t st) {
  size_t need = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, need, inout, inout, (int)n_plus_1, st);
  if (need > ws_bytes) return FS_ECAPACITY;
  FS_CUDA_CHECK(cub::DeviceScan::ExclusiveSum(ws, need, inout, inout, (int)n_plus_1, st));
  return FS_OK;
}

int launch_node_offsets(const fs_pose_batch& b, int64_t* node_off, void* ws, size_t ws_bytes,
                        cudaStream_t st, int64_t clamp) {
  if (b.n_poses <= 0) return cuda_status(cudaMemsetAsync(node_off, 0, sizeof(int64_t), st));
  pose_node_counts_kernel<<<(int)cdiv(b.n_poses, 256), 256, 0, st>>>(b, node_off, clamp);
  FS_LAUNCH_CHECK();
  FS_CUDA_CHECK(cudaMemsetAsync(node_off + b.n_poses, 0, sizeof(int64_t), st));
  return exclusive_scan_i64(node_off, b.n_poses + 1, ws, ws_bytes, st);
}

int launch_voxelize(const fs_pose_batch& b, int g, int c_elem, double box, int layout, void* out,
                    int32_t* err, cudaStream_t st) {
  if (g < 8) return FS_EINVAL;                     // complexes.py:149-151
  if (b.n_poses <= 0) return FS_OK;
  VoxParams v;
  v.g = g; v.c_elem = c_elem; v.channels = 2 * c_elem; v.layout = layout;
  v.half = box / 2.0; v.box = box; v.gd = (double)g;
  const int64_t cells = (int64_t)v.channels * g * g * g;
  const size_t smem = (size_t)cells * 4;
  if (layout == FS_GRID_NDHWC_BF16 && v.channels % 8 == 0 && cells * 2 <= 200 * 1024 &&
      b.max_pose_atoms > 0 && b.max_pose_atoms < 65536) {
    const size_t sm2 = (size_t)cells * 2;
    FS_CUDA_CHECK(cudaFuncSetAttribute(voxelize_bf16_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm2));
    voxelize_bf16_kernel<<<b.n_poses, 512, sm2, st>>>(b, v, (__nv_bfloat16*)out, err);
  } else if (smem <= 200 * 1024) {
    FS_CUDA_CHECK(cudaFuncSetAttribute(voxelize_smem_kernel,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    voxelize_smem_kernel<<<b.n_poses, 512, smem, st>>>(b, v, out, err);
  } else {
    if (layout == FS_GRID_NDHWC_BF16) return FS_ENOTSUP;
    size_t es = layout == FS_GRID_NCDHW_F64 ? 8 : 4;
    FS_CUDA_CHECK(cudaMemsetAsync(out, 0, es * cells * b.n_poses, st));
    voxelize_global_kernel<<<b.n_poses, 256, 0, st>>>(b, v, out, err);
  }
  FS_LAUNCH_CHECK();
  return FS_OK;
}

int launch_node_features(const fs_pose_batch& b, const int64_t* node_off, int c_elem, double box,
                         void* out, bool f64, cudaStream_t st) {
  if (b.n_poses <= 0) return FS_OK;
  if (f64) node_features_kernel<double><<<b.n_poses, 256, 0, st>>>(b, node_off, c_elem, box, (double*)out);
  else node_features_kernel<float><<<b.n_poses, 256, 0, st>>>(b, node_off, c_elem, box, (float*)out);
  FS_LAUNCH_CHECK();
  return FS_OK;
}

static int graph_smem_atoms(const fs_pose_batch& b) {
  int m = b.max_pose_atoms > 0 ? b.max_pose_atoms : FS_MAX_POSE_ATOMS;
  return m > FS_MAX_POSE_ATOMS ? FS_MAX_POSE_ATOMS : m;
}

int launch_graph_count(const fs_pose_batch& b, const int64_t* node_off, double tc, double tn,
                       int32_t* deg_cov, int32_t* deg_ncov, int32_t* err, cudaStream_t st) {
  if (!(tc >= 1.2 && tc <= 5.9) || !(tn >= 1.2 && tn <= 5.9)) return FS_EINVAL;  // complexes.py:228-231
  if (b.n_poses <= 0) return FS_OK;
  const int atoms = graph_smem_atoms(b);
  const size_t smem = graph_smem_bytes(atoms);
  FS_CUDA_CHECK(cudaFuncSetAttribute(graph_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  graph_kernel<false><<<b.n_poses, kGraphThreads, smem, st>>>(
      b, node_off, tc, tn, deg_cov, deg_ncov, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr,
      0, 0, err, atoms);
  FS_LAUNCH_CHECK();
  return FS_OK;
}

int launch_graph_fill(const fs_pose_batch& b, const int64_t* node_off, double tc, double tn,
                      const int64_t* row_cov, const int64_t* row_ncov, int32_t* col_cov,
                      int32_t* col_ncov, double* dist_cov, double* dist_ncov, int64_t cap_cov,
                      int64_t cap_ncov, int32_t* err, cudaStream_t st) {
  if (!(tc >= 1.2 && tc <= 5.9) || !(tn >= 1.2 && tn <= 5.9)) return FS_EINVAL;
  if (b.n_poses <= 0) return FS_OK;
  const int atoms = graph_smem_atoms(b);
  const size_t smem = graph_smem_bytes(atoms);
  FS_CUDA_CHECK(cudaFuncSetAttribute(graph_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  graph_kernel<true><<<b.n_poses, kGraphThreads, smem, st>>>(
      b, node_off, tc, tn, nullptr, nullptr, row_cov, row_ncov, col_cov, col_ncov, dist_cov,
      dist_ncov, cap_cov, cap_ncov, err, atoms);
  FS_LAUNCH_CHECK();
  return FS_OK;
}

int launch_rows(const int32_t* deg, int64_t n, int64_t* row_ptr, void* ws, size_t ws_bytes,
                cudaStream_t st) {
  widen_kernel<<<(int)cdiv(n + 1, 256), 256, 0, st>>>(deg, n, row_ptr);
  FS_LAUNCH_CHECK();
  return exclusive_scan_i64(row_ptr, n + 1, ws, ws_bytes, st);
}

int launch_edge_counts(const int64_t* node_off, int n_poses, const int64_t* row_ptr,
                       const int32_t* col, int64_t* edge_off, void* ws, size_t ws_bytes,
                       cudaStream_t st) {
  if (n_poses <= 0) return cuda_status(cudaMemsetAsync(edge_off, 0, 8, st));
  upper_counts_kernel<<<n_poses, 256, 0, st>>>(node_off, n_poses, row_ptr, col, edge_off);
  FS_LAUNCH_CHECK();
  FS_CUDA_CHECK(cudaMemsetAsync(edge_off + n_poses, 0, 8, st));
  return exclusive_scan_i64(edge_off, n_poses + 1, ws, ws_bytes, st);
}

int launch_edges(const int64_t* node_off, int n_poses, const int64_t* row_ptr, const int32_t* col,
                 const double* dist, const int64_t* edge_off, int64_t* edges, double* dists,
                 cudaStream_t st) {
  if (n_poses <= 0) return FS_OK;
  upper_edges_kernel<<<n_poses, 32, 0, st>>>(node_off, n_poses, row_ptr, col, dist, edge_off, edges, dists);
  FS_LAUNCH_CHECK();
  return FS_OK;
}

// Symmetric CSR from i<j global edge list.  deg is [n] int32 scratch,
// cursor [n+1] int64 scratch.
int launch_csr_from_edges(const int64_t* edges, int64_t ne, const int64_t* node_off, int n_poses,
                          int64_t n_nodes, int32_t* node_pose, int32_t* deg, int64_t* row_ptr,
                          int64_t* cursor, col_t* col, void* ws, size_t ws_bytes, cudaStream_t st) {
  if (n_nodes <= 0) return FS_OK;
  node_pose_kernel<<<n_poses, 256, 0, st>>>(node_off, n_poses, node_pose);
  FS_LAUNCH_CHECK();
  FS_CUDA_CHECK(cudaMemsetAsync(deg, 0, sizeof(int32_t) * n_nodes, st));
  if (ne > 0) {
    edge_degree_kernel<<<(int)cdiv(ne, 256), 256, 0, st>>>(edges, ne, deg);
    FS_LAUNCH_CHECK();
  }
  int rc = launch_rows(deg, n_nodes, row_ptr, ws, ws_bytes, st);
  if (rc) return rc;
  if (ne > 0) {
    FS_CUDA_CHECK(cudaMemcpyAsync(cursor, row_ptr, sizeof(int64_t) * (n_nodes + 1),
                                  cudaMemcpyDeviceToDevice, st));
    edge_fill_kernel<<<(int)cdiv(ne, 256), 256, 0, st>>>(edges, ne, node_off, node_pose, cursor, col);
    FS_LAUNCH_CHECK();
    sort_rows_kernel<<<(int)cdiv(n_nodes, 256), 256, 0, st>>>(row_ptr, n_nodes, col);
    FS_LAUNCH_CHECK();
  }
  return FS_OK;
}

}  // namespace fs
