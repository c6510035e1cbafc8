// Fused single-launch radius graph for the scoring path: one CTA per pose
// builds both CSR adjacencies (covalent / non-covalent) of its pose in a
// private slice [p*cap, (p+1)*cap) of the column arrays.  Same exact edge
// predicate as featurize.cu (complexes.py:237-246):
//   d2 = (dx*dx+dy*dy)+dz*dz (float64, no FMA); candidate iff d2 <= rmax^2;
//   keep iff sqrt(d2) <= t_cov (same role) / t_ncov (different role).
// Rows are written as (start, deg); non-covalent rows ascend in the neighbour
// id, covalent rows do when distances are requested (see the fill below).
//
// Work split:
//  * non-covalent pairs are bipartite (role S x role L, S the smaller role):
//    each warp scans one S atom against the L list 32 candidates at a time
//    (index-ascending, ballot-compacted) and sets bit s in an L-row bitmask.
//    Every S-L pair is tested exactly once; L rows are read back from the
//    masks in ascending S order (the S list is index-sorted).
//  * covalent pairs: cell list with cells >= t_cov (27-cell stencil), one
//    thread per row, counted then filled and insertion-sorted.
//  * all scans are parallel (no serial per-cell loops).
#include "common.cuh"

namespace fs {

struct GraphCsrArgs {
  fs_pose_batch b;
  const int64_t* node_off;
  double tc, tn;
  int64_t* row_cov; int32_t* deg_cov; col_t* col_cov; double* dist_cov;
  int64_t* row_ncov; int32_t* deg_ncov; col_t* col_ncov; double* dist_ncov;
  int64_t cap;          // entries per pose per edge type
  int32_t* err;
  int smem_atoms;
  float* feats;         // optional node features [N][c_elem + 4] (node_features_kernel<float>)
  int c_elem; double box;
};

#ifndef FS_CELLS_AXIS
#define FS_CELLS_AXIS 9
#endif
constexpr int kCsrThreads = 256;
constexpr int kCsrWarps = kCsrThreads / 32;
constexpr int kCellsAxis = FS_CELLS_AXIS;   // cells grow past t_cov for boxes > kCellsAxis * t_cov
constexpr int kMaskWords = 2;         // bipartite bitmask path for |S| <= 64
constexpr int kCovBits = 96;          // covalent candidates per row whose hit bits are kept
constexpr int kCovWords = kCovBits / 32;
constexpr int kCellWords = 2 * kCellsAxis * kCellsAxis * kCellsAxis + 2;

// 46 bytes per atom + cell table: <= 55.75 KB at the workload's 1,064 atoms,
// so four 256-thread CTAs share an SM (three at the former 74 KB)
__host__ __device__ inline size_t graph_csr_smem_bytes(int n) {
  n = (n + 3) & ~3;   // keeps every sub-array 8-byte aligned
  return (size_t)n * 16 + (size_t)n * 2 * 5 + (size_t)n * kMaskWords * 4 + (size_t)kCellWords * 4 +
         (size_t)n * kCovWords * 4 + (size_t)(n + 31) / 32 * 4 + 16;
}

// 32x32 bit-matrix transpose across a warp: on return, bit j of lane l is
// bit l of lane j's input (one row index bit swapped with one column index
// bit per butterfly stage)
__device__ __forceinline__ uint32_t warp_transpose32(uint32_t x, int lane) {
  constexpr uint32_t kLow[5] = {0x0000FFFFu, 0x00FF00FFu, 0x0F0F0F0Fu, 0x33333333u, 0x55555555u};
#pragma unroll
  for (int k = 0; k < 5; ++k) {
    const int s = 16 >> k;
    const bool upper = lane & s;
    const uint32_t keep = upper ? ~kLow[k] : kLow[k];
    const uint32_t out = x & ~keep;
    const uint32_t y = __shfl_xor_sync(0xffffffffu, upper ? out << s : out >> s, s);
    x = (x & keep) | y;
  }
  return x;
}

// Exclusive scan of u16 counts c[0..n) into out[i] = base + prefix (int64,
// global); returns the total.  Starts with a barrier.
__device__ int block_scan_u16_to_global(const uint16_t* c, int n, int64_t* out, int64_t base, int* warp_tot) {
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int per = (n + blockDim.x - 1) / blockDim.x;
  const int lo = min(n, (int)threadIdx.x * per), hi = min(n, lo + per);
  int sum = 0;
  for (int i = lo; i < hi; ++i) sum += c[i];
  int incl = sum;
  for (int o = 1; o < 32; o <<= 1) {
    int v = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += v;
  }
  if (lane == 31) warp_tot[warp] = incl;
  __syncthreads();
  if (threadIdx.x == 0) {
    int run = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) { int v = warp_tot[w]; warp_tot[w] = run; run += v; }
    warp_tot[31] = run;
  }
  __syncthreads();
  int run = warp_tot[warp] + incl - sum;
  for (int i = lo; i < hi; ++i) { out[i] = base + run; run += c[i]; }
  const int tot = warp_tot[31];
  __syncthreads();
  return tot;
}

// in-place exclusive scan of a[0..n) (n+1-th entry receives the total).
// Starts with a barrier: the caller's writes to a[] are visible to every thread.
__device__ void block_exclusive_scan(int* a, int n, int* warp_tot) {
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int per = (n + blockDim.x - 1) / blockDim.x;
  const int lo = min(n, (int)threadIdx.x * per), hi = min(n, lo + per);
  int sum = 0;
  for (int i = lo; i < hi; ++i) sum += a[i];
  int incl = sum;
  for (int o = 1; o < 32; o <<= 1) {
    int v = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += v;
  }
  if (lane == 31) warp_tot[warp] = incl;
  __syncthreads();
  if (threadIdx.x == 0) {
    int run = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) { int v = warp_tot[w]; warp_tot[w] = run; run += v; }
    warp_tot[31] = run;
  }
  __syncthreads();
  int run = warp_tot[warp] + incl - sum;
  for (int i = lo; i < hi; ++i) { int v = a[i]; a[i] = run; run += v; }
  __syncthreads();
  if (threadIdx.x == 0) a[n] = warp_tot[31];
  __syncthreads();
}

// exact float64 predicate; coordinates come from global memory (the fp32
// band test makes this path rare on the scoring path)
__device__ __forceinline__ bool exact_edge(const PoseView& pv, double xi, double yi, double zi, int j,
                                           double rmax2, double t, double* dout) {
  double xj, yj, zj; int32_t ej, rj;
  pv.atom(j, xj, yj, zj, ej, rj);
  const double d2 = dist2_exact(xi - xj, yi - yj, zi - zj);
  if (!(d2 <= rmax2)) return false;
  const double d = __dsqrt_rn(d2);
  if (!(d <= t)) return false;
  *dout = d;
  return true;
}

// Out-of-line copy for the in-band case of the fp32 decision: keeps the fp64
// code out of the hot candidate loops (inlined, it would be predicated into
// every iteration).
__device__ __noinline__ bool exact_edge_slow(PoseView pv, double xi, double yi, double zi, int j, double rmax2,
                                             double t) {
  double d;
  return exact_edge(pv, xi, yi, zi, j, rmax2, t, &d);
}

// exact predicate for the pair (i, j) with i's coordinates first (the
// bipartite scans' S - L order), out of line like exact_edge_slow
__device__ __noinline__ bool exact_pair_slow(PoseView pv, int i, int j, double rmax2, double t) {
  double xi, yi, zi; int32_t e, r;
  pv.atom(i, xi, yi, zi, e, r);
  double d;
  return exact_edge(pv, xi, yi, zi, j, rmax2, t, &d);
}

template <bool DIST>
__global__ void __launch_bounds__(kCsrThreads) graph_csr_kernel(GraphCsrArgs a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ double red[33];
  __shared__ double s_min[3];
  __shared__ int s_flags, s_n0;
  __shared__ int warp_tot[32];
  __shared__ int warp_cnt[kCsrWarps];

  const int p = blockIdx.x;
  const PoseView pv = pose_view(a.b, p);
  const int n = (int)pv.n();
  const int64_t base = a.node_off[p];
  const int64_t cbase = (int64_t)p * a.cap;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;

  auto fail = [&](int flags) {
    if (threadIdx.x == 0) atomicOr(&a.err[p], flags);
    // an oversize pose owns only smem_atoms node rows (launch_node_offsets
    // clamps its count), so empty rows are written for those alone
    const int nr = min(n, a.smem_atoms);
    for (int i = threadIdx.x; i < nr; i += blockDim.x) {
      a.deg_cov[base + i] = 0; a.deg_ncov[base + i] = 0;
      a.row_cov[base + i] = cbase; a.row_ncov[base + i] = cbase;
    }
  };
  if (threadIdx.x == 0) s_flags = 0;
  if (n > a.smem_atoms) { fail(FS_ERR_TOO_LARGE); return; }
  const int SA = (a.smem_atoms + 3) & ~3;   // 16-byte aligned sub-arrays
  float4* pf = reinterpret_cast<float4*>(smem_raw);
  uint16_t* keys = reinterpret_cast<uint16_t*>(pf + SA);   // (role, cell) key < 2^16
  uint16_t* cell_list = keys + SA;      // atoms in (role, cell) order (first: role ranks)
  uint16_t* role_list = cell_list + SA; // role 0 ids ascending, then role 1 ids ascending
  uint16_t* offc = role_list + SA;      // covalent degree per row (row starts live in row_cov)
  uint16_t* offn = offc + SA;           // non-covalent degree per row
  uint32_t* mask = reinterpret_cast<uint32_t*>(offn + SA);   // [|L|][kMaskWords]
  int* cell_start = reinterpret_cast<int*>(mask + (size_t)SA * kMaskWords);
  uint32_t* covbits = reinterpret_cast<uint32_t*>(cell_start + kCellWords);   // [n][kCovWords]
  uint32_t* ovf = covbits + (size_t)SA * kCovWords;   // rows whose hit bits do not cover their candidates
  __syncthreads();

  // ---- atoms, validation, bounding box ----
  double lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
  int flags = 0;
  float* fo = a.feats ? a.feats + base * (a.c_elem + 4) : nullptr;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    double x, y, z; int32_t e, r;
    pv.atom(i, x, y, z, e, r);
    if (fo) {   // node features (complexes.py:233-236), as node_features_kernel<float>
      const int F = a.c_elem + 4, ec = min(max(e, 0), a.c_elem - 1);
      float* f = fo + (int64_t)i * F;
      for (int c = 0; c < a.c_elem; ++c) f[c] = c == ec ? 1.f : 0.f;
      f[a.c_elem] = (float)r;
      f[a.c_elem + 1] = (float)__dadd_rn(__ddiv_rn(x, a.box), 0.5);
      f[a.c_elem + 2] = (float)__dadd_rn(__ddiv_rn(y, a.box), 0.5);
      f[a.c_elem + 3] = (float)__dadd_rn(__ddiv_rn(z, a.box), 0.5);
    }
    if (r != 0 && r != 1) flags |= FS_ERR_ROLE;
    if (!isfinite(x) || !isfinite(y) || !isfinite(z)) flags |= FS_ERR_NONFINITE;
    pf[i] = make_float4((float)x, (float)y, (float)z, (float)r);
    lo[0] = fmin(lo[0], x); lo[1] = fmin(lo[1], y); lo[2] = fmin(lo[2], z);
    hi[0] = fmax(hi[0], x); hi[1] = fmax(hi[1], y); hi[2] = fmax(hi[2], z);
  }
  if (flags) atomicOr(&s_flags, flags);
  // the six bounds in one block reduction (fmin / fmax are order-free),
  // through the cell table (zeroed only after it)
  double ext_max = 0.0, absmax = 0.0;
  {
    double* rb = reinterpret_cast<double*>(cell_start);   // [6][kCsrWarps]
#pragma unroll
    for (int ax = 0; ax < 3; ++ax) {
      for (int o = 16; o > 0; o >>= 1) {
        lo[ax] = fmin(lo[ax], __shfl_xor_sync(0xffffffffu, lo[ax], o));
        hi[ax] = fmax(hi[ax], __shfl_xor_sync(0xffffffffu, hi[ax], o));
      }
      if (lane == 0) { rb[ax * kCsrWarps + warp] = lo[ax]; rb[(3 + ax) * kCsrWarps + warp] = hi[ax]; }
    }
    __syncthreads();
#pragma unroll
    for (int ax = 0; ax < 3; ++ax) {
      double l = rb[ax * kCsrWarps], h = rb[(3 + ax) * kCsrWarps];
      for (int w = 1; w < kCsrWarps; ++w) { l = fmin(l, rb[ax * kCsrWarps + w]); h = fmax(h, rb[(3 + ax) * kCsrWarps + w]); }
      if (threadIdx.x == 0) s_min[ax] = l;
      ext_max = fmax(ext_max, h - l);
      absmax = fmax(absmax, fmax(fabs(l), fabs(h)));
    }
  }
  __syncthreads();
  if (s_flags) { fail(s_flags); return; }
  if (n == 0) return;
  const bool prefilter = absmax < 1024.0;            // fp32 coordinate error <= 6.1e-5 A
  // cells >= 1.001 t_cov: the fp32 cell index below (coordinate error
  // <= 6.1e-5 A when |x| < 1024) cannot separate a covalent pair by two cells
  const double cs = fmax(a.tc * 1.001, ext_max / (kCellsAxis - 1));
  const int nca = min(kCellsAxis, (int)floor(ext_max / cs) + 1);
  const int NC = nca * nca * nca;
  for (int i = threadIdx.x; i < 2 * NC + 1; i += blockDim.x) cell_start[i] = 0;
  __syncthreads();
  auto cell_coord = [&](double x, int ax) -> int {
    int c = (int)floor(__ddiv_rn(__dsub_rn(x, s_min[ax]), cs));
    return min(max(c, 0), nca - 1);
  };
  const float inv_cs = (float)(1.0 / cs);
  const float fmin_x = (float)s_min[0], fmin_y = (float)s_min[1], fmin_z = (float)s_min[2];
  auto cell_coord_f = [&](float x, float m) -> int {
    const int c = (int)floorf((x - m) * inv_cs);
    return min(max(c, 0), nca - 1);
  };

  // ---- counting sort by (role, cell); role lists ascending by id ----
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const float4 f = pf[i];
    const int r = (int)f.w;
    int cx, cy, cz;
    if (prefilter) {
      cx = cell_coord_f(f.x, fmin_x); cy = cell_coord_f(f.y, fmin_y); cz = cell_coord_f(f.z, fmin_z);
    } else {
      double x, y, z; int32_t e, rr;
      pv.atom(i, x, y, z, e, rr);
      cx = cell_coord(x, 0); cy = cell_coord(y, 1); cz = cell_coord(z, 2);
    }
    // keys hold (role, cx, cy, cz) packed in 4-bit fields (nca <= 9): the
    // stencil loops decompose them with shifts instead of divisions
    keys[i] = (uint16_t)(r << 12 | cx << 8 | cy << 4 | cz);
    atomicAdd(&cell_start[r * NC + (cx * nca + cy) * nca + cz], 1);
  }
  // role lists: each thread takes a contiguous id range; one block scan of
  // the role-0 counts places every id (roles are 0 / 1, validated above)
  {
    const int per = (n + blockDim.x - 1) / blockDim.x;
    const int i0 = min(n, (int)threadIdx.x * per), i1 = min(n, i0 + per);
    int c = 0;
    for (int i = i0; i < i1; ++i) c += pf[i].w == 0.f;
    int inc = c;
    for (int o = 1; o < 32; o <<= 1) {
      const int v = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += v;
    }
    if (lane == 31) warp_cnt[warp] = inc;
    __syncthreads();
    int before = 0, tot = 0;
    for (int w = 0; w < kCsrWarps; ++w) { const int v = warp_cnt[w]; before += w < warp ? v : 0; tot += v; }
    if (threadIdx.x == 0) s_n0 = tot;
    int p0 = before + inc - c, p1 = tot + i0 - p0;   // this range's first role-0 / role-1 slots
    for (int i = i0; i < i1; ++i) role_list[pf[i].w == 0.f ? p0++ : p1++] = (uint16_t)i;
  }
  block_exclusive_scan(cell_start, 2 * NC, warp_tot);
  const int n0 = s_n0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const int kp = keys[i];
    const int slot = atomicAdd(&cell_start[(kp >> 12) * NC + (((kp >> 8) & 15) * nca + ((kp >> 4) & 15)) * nca +
                                           (kp & 15)], 1);   // becomes the cell end
    FS_DCHECK(slot < n, "graph cell slot", slot, n);
    cell_list[slot] = (uint16_t)i;
  }
  __syncthreads();
  // cell k spans [cell_start[k-1], cell_start[k]) now (cell_start[-1] := 0);
  // sort each (few-atom) cell by id so the candidate order is deterministic
  for (int k = threadIdx.x; k < 2 * NC; k += blockDim.x) {
    const int cb = k == 0 ? 0 : cell_start[k - 1], ce = cell_start[k];
    for (int x = cb + 1; x < ce; ++x) {
      const uint16_t v = cell_list[x];
      int y = x - 1;
      while (y >= cb && cell_list[y] > v) { cell_list[y + 1] = cell_list[y]; --y; }
      cell_list[y + 1] = v;
    }
  }
  __syncthreads();

  const double rmax = fmax(a.tc, a.tn);
  const double rmax2 = __dmul_rn(rmax, rmax);
  // fp32 decision band.  With |coords| <= M the fp32 distance differs from
  // the float64 one by < 2^-21*M + 4 ulp; outside [t - delta, t + delta] the
  // fp32 test decides exactly, inside it the float64 predicate runs.
  const float delta = 1e-5f + 2e-6f * (float)absmax;
  // Without the prefilter (|coords| >= 1024 A) the band is everything: every
  // pair takes the exact path, with no per-candidate prefilter test.
  const float c_lo2 = prefilter ? ((float)a.tc - delta) * ((float)a.tc - delta) : -1.0f;
  const float c_hi2 = prefilter ? ((float)a.tc + delta) * ((float)a.tc + delta) : INFINITY;
  const float n_lo2 = prefilter ? ((float)a.tn - delta) * ((float)a.tn - delta) : -1.0f;
  const float n_hi2 = prefilter ? ((float)a.tn + delta) * ((float)a.tn + delta) : INFINITY;
  // covalent band as centre / half-width (a slightly wider band; without the
  // prefilter every candidate is in it)
  const float c_mid2 = prefilter ? 0.5f * (c_lo2 + c_hi2) : 0.0f;
  const float c_half2 = prefilter ? 0.5f * (c_hi2 - c_lo2) * 1.0001f + 1e-6f : INFINITY;
  const float n_mid2 = prefilter ? 0.5f * (n_lo2 + n_hi2) : 0.0f;
  const float n_half2 = prefilter ? 0.5f * (n_hi2 - n_lo2) * 1.0001f + 1e-6f : INFINITY;
  // 1: edge, 0: not, decided in fp32; inside the band the exact float64 predicate
  auto decide = [&](float d2f, float lo2, float hi2, double xi, double yi, double zi, int j, double t) -> bool {
    if (d2f > hi2) return false;
    if (d2f <= lo2) return true;
    double d;
    return exact_edge(pv, xi, yi, zi, j, rmax2, t, &d);
  };
  // same, loading row i's float64 coordinates only inside the band
  auto decide_i = [&](float d2f, float lo2, float hi2, int i, int j, double t) -> bool {
    if (d2f > hi2) return false;
    if (d2f <= lo2) return true;
    double xi, yi, zi; int32_t e_, r_;
    pv.atom(i, xi, yi, zi, e_, r_);
    double d;
    return exact_edge(pv, xi, yi, zi, j, rmax2, t, &d);
  };

  // ---- non-covalent: bipartite S x L ----
  const int n1 = n - n0;
  const int sr = n0 <= n1 ? 0 : 1;                 // smaller role
  const int nS = sr == 0 ? n0 : n1, nL = n - nS;
  const uint16_t* Slist = role_list + (sr == 0 ? 0 : n0);
  const uint16_t* Llist = role_list + (sr == 0 ? n0 : 0);
  const bool use_mask = nS <= 32 * kMaskWords;
  const int W = (nS + 31) / 32;
  for (int i = threadIdx.x; i < n; i += blockDim.x) { offc[i] = 0; offn[i] = 0; }
  for (int i = threadIdx.x; i < (n + 31) / 32; i += blockDim.x) ovf[i] = 0u;
  if (use_mask) {
    // lanes over L atoms (32 per warp chunk), loop over the S atoms (broadcast
    // shared reads): the chunk's per-S-atom ballots become the L rows' hit
    // masks (no atomics on the mask); S-row counts accumulate per lane.  The
    // masks are the only record of the decisions: both fills read them.
    int* s_ncnt = reinterpret_cast<int*>(red);   // [<= 64], red is free here
    if (threadIdx.x < 32 * kMaskWords) s_ncnt[threadIdx.x] = 0;
    __syncthreads();
    int sacc0 = 0, sacc1 = 0;   // lane l: hits of S atoms l and 32 + l in this warp's chunks
    for (int l0 = warp * 32; l0 < nL; l0 += kCsrWarps * 32) {
      const int lj = l0 + lane;
      const bool lv = lj < nL;
      const int j = lv ? Llist[lj] : 0;
      // idle lanes sit at infinity: never a hit, never in the band
      const float4 fj = lv ? pf[j] : make_float4(INFINITY, INFINITY, INFINITY, 0.f);
      // lane l keeps the chunk's ballot of S atom l (b0) / 32 + l (b1) of the
      // fp32-certain hits; one warp transpose per word turns them into the L
      // rows' masks.  The band test is one distance to the band's middle (a
      // superset); a lane that saw the band settles its row exactly below.
      uint32_t b0 = 0u, b1 = 0u;
      float bmin = INFINITY;
      auto sweep = [&](int s0, int s1, uint32_t& bw) {
#pragma unroll 4
        for (int si = s0; si < s1; ++si) {
          const float4 fi = pf[Slist[si]];
          const float dx = fi.x - fj.x, dy = fi.y - fj.y, dz = fi.z - fj.z;
          const float d2f = dx * dx + dy * dy + dz * dz;
          bmin = fminf(bmin, fabsf(d2f - n_mid2));
          const uint32_t bal = __ballot_sync(0xffffffffu, d2f <= n_lo2);
          bw = lane == si - s0 ? bal : bw;
        }
      };
      sweep(0, min(nS, 32), b0);
      if (nS > 32) sweep(32, nS, b1);
      uint32_t m0 = warp_transpose32(b0, lane);
      uint32_t m1 = W > 1 ? warp_transpose32(b1, lane) : 0u;
      const bool band = bmin <= n_half2;
      if (__any_sync(0xffffffffu, band)) {   // rare: exact float64 predicate inside the band
        if (band) {
          for (int si = 0; si < nS; ++si) {
            const int i = Slist[si];
            const float4 fi = pf[i];
            const float dx = fi.x - fj.x, dy = fi.y - fj.y, dz = fi.z - fj.z;
            const float d2f = dx * dx + dy * dy + dz * dz;
            if (lv && d2f > n_lo2 && d2f <= n_hi2 && exact_pair_slow(pv, i, j, rmax2, a.tn)) {
              if (si < 32) m0 |= 1u << si;
              else m1 |= 1u << (si - 32);
            }
          }
        }
        b0 = warp_transpose32(m0, lane);
        if (W > 1) b1 = warp_transpose32(m1, lane);
      }
      sacc0 += __popc(b0);
      sacc1 += __popc(b1);
      if (lv) {
        mask[lj * W] = m0;
        if (W > 1) mask[lj * W + 1] = m1;
        offn[j] = (uint16_t)(__popc(m0) + __popc(m1));
      }
    }
    if (sacc0) atomicAdd(&s_ncnt[lane], sacc0);
    if (sacc1) atomicAdd(&s_ncnt[32 + lane], sacc1);
    __syncthreads();
    for (int si = threadIdx.x; si < nS; si += blockDim.x) offn[Slist[si]] = (uint16_t)s_ncnt[si];
  } else {
    // large bipartite sides: one thread per row scans the other role's list
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
      double xi, yi, zi; int32_t ei_, ri_; pv.atom(i, xi, yi, zi, ei_, ri_);
      const float4 fi = pf[i];
      const int ri = (int)fi.w;
      const int ob = ri == 0 ? n0 : 0, oe = ri == 0 ? n : n0;
      int c = 0;
      for (int q = ob; q < oe; ++q) {
        const int j = role_list[q];
        const float4 fj = pf[j];
        const float dx = fi.x - fj.x, dy = fi.y - fj.y, dz = fi.z - fj.z;
        c += decide(dx * dx + dy * dy + dz * dz, n_lo2, n_hi2, xi, yi, zi, j, a.tn);
      }
      offn[i] = c;
    }
  }

  // ---- covalent degrees: 27-cell stencil, one thread per row ----
  auto cov_scan = [&](int i, auto&& emit) {
    double xi, yi, zi; int32_t ei_, ri_; pv.atom(i, xi, yi, zi, ei_, ri_);
    const float4 fi = pf[i];
    const int ri = (int)fi.w;
    const int kp = keys[i];
    const int cz = kp & 15, cy = (kp >> 4) & 15, cx = (kp >> 8) & 15;
    for (int dx = -1; dx <= 1; ++dx) {
      const int ax = cx + dx;
      if (ax < 0 || ax >= nca) continue;
      for (int dy = -1; dy <= 1; ++dy) {
        const int ay = cy + dy;
        if (ay < 0 || ay >= nca) continue;
        // the three z-neighbour cells are contiguous in cell order
        const int z0 = max(cz - 1, 0), z1 = min(cz + 1, nca - 1);
        const int k0 = ri * NC + (ax * nca + ay) * nca + z0, k1 = ri * NC + (ax * nca + ay) * nca + z1;
        const int qb = k0 == 0 ? 0 : cell_start[k0 - 1], qe = cell_start[k1];
        for (int q = qb; q < qe; ++q) {
          const int j = cell_list[q];
          if (j == i) continue;
          const float4 fj = pf[j];
          const float ddx = fi.x - fj.x, ddy = fi.y - fj.y, ddz = fi.z - fj.z;
          if (decide(ddx * ddx + ddy * ddy + ddz * ddz, c_lo2, c_hi2, xi, yi, zi, j, a.tc)) emit(j);
        }
      }
    }
  };
  // count pass: the hit pattern over the first kCovBits candidates is kept
  // (covbits) so the fill pass emits without re-testing distances
  // rows are taken in cell order: a warp's rows share their stencil cells
  // (same trip counts, broadcast candidate reads)
  for (int idx = threadIdx.x; idx < n; idx += blockDim.x) {
    const int i = cell_list[idx];
    const float4 fi = pf[i];
    int cnt = 0, c0 = 0;
    bool over = false;
    uint32_t w0 = 0u, w1 = 0u, w2 = 0u;   // hit bits of candidates 0..95
    const int ri = (int)fi.w;
    const int kp = keys[i];
    const int cz = kp & 15, cy = (kp >> 4) & 15, cx = (kp >> 8) & 15;
    for (int dx = -1; dx <= 1; ++dx) {
      const int ax = cx + dx;
      if (ax < 0 || ax >= nca) continue;
      for (int dy = -1; dy <= 1; ++dy) {
        const int ay = cy + dy;
        if (ay < 0 || ay >= nca) continue;
        const int z0 = max(cz - 1, 0), z1 = min(cz + 1, nca - 1);
        const int k0 = ri * NC + (ax * nca + ay) * nca + z0, k1 = ri * NC + (ax * nca + ay) * nca + z1;
        const int qb = k0 == 0 ? 0 : cell_start[k0 - 1], qe = cell_start[k1];
        // one stencil column: hits collected run-locally, merged once.  The
        // row's own atom is a candidate here (it always hits: d = 0); the
        // count drops it at the end and the fill never emits it.
        uint64_t rm = 0ull;
        const int len = qe - qb;
        if (len <= 64) {
          // branch-free candidate loop: fp32-certain hits as a bit set (32-bit
          // for the usual short column), one in-band flag; the (rare) band is
          // settled exactly afterwards
          bool anyband = false;
          if (len <= 32) {
            // hits shifted in from the top (bit k <- candidate qe-1-k..), one
            // reversal after the loop; the band test as one distance to the
            // band's middle (a superset of the band: the re-walk is exact)
            uint32_t r32 = 0u;
            float bmin = INFINITY;
            for (int q = qb; q < qe; ++q) {
              const int j = cell_list[q];
              const float4 fj = pf[j];
              const float ddx = fi.x - fj.x, ddy = fi.y - fj.y, ddz = fi.z - fj.z;
              const float d2f = ddx * ddx + ddy * ddy + ddz * ddz;
              r32 = (r32 >> 1) | (d2f <= c_lo2 ? 0x80000000u : 0u);
              bmin = fminf(bmin, fabsf(d2f - c_mid2));
            }
            rm = len ? r32 >> (32 - len) : 0u;
            anyband = bmin <= c_half2;
          } else {
            for (int q = qb; q < qe; ++q) {
              const int j = cell_list[q];
              const float4 fj = pf[j];
              const float ddx = fi.x - fj.x, ddy = fi.y - fj.y, ddz = fi.z - fj.z;
              const float d2f = ddx * ddx + ddy * ddy + ddz * ddz;
              rm |= (uint64_t)(d2f <= c_lo2) << (q - qb);
              anyband |= d2f > c_lo2 && d2f <= c_hi2;
            }
          }
          if (anyband) {   // rare: re-walk the column, settle in-band pairs exactly
            for (int q = qb; q < qe; ++q) {
              const int j = cell_list[q];
              const float4 fj = pf[j];
              const float ddx = fi.x - fj.x, ddy = fi.y - fj.y, ddz = fi.z - fj.z;
              const float d2f = ddx * ddx + ddy * ddy + ddz * ddz;
              if (d2f > c_lo2 && d2f <= c_hi2 && decide_i(c_lo2 + 1.0f, c_lo2, INFINITY, i, j, a.tc))
                rm |= 1ull << (q - qb);
            }
          }
        } else {   // crowded column: counted only, the fill re-tests this row
          over = true;
          for (int q = qb; q < qe; ++q) {
            const int j = cell_list[q];
            const float4 fj = pf[j];
            const float ddx = fi.x - fj.x, ddy = fi.y - fj.y, ddz = fi.z - fj.z;
            cnt += decide_i(ddx * ddx + ddy * ddy + ddz * ddz, c_lo2, c_hi2, i, j, a.tc);
          }
        }
        cnt += __popcll(rm);
        if (c0 < kCovBits) {
          const int sh = c0 & 31;
          const uint64_t x = rm << sh;
          const uint32_t p0 = (uint32_t)x, p1 = (uint32_t)(x >> 32), p2 = sh ? (uint32_t)(rm >> (64 - sh)) : 0u;
          if (c0 < 32) { w0 |= p0; w1 |= p1; w2 |= p2; }
          else if (c0 < 64) { w1 |= p0; w2 |= p1; }
          else { w2 |= p0; }
        }
        c0 += len;
      }
    }
    uint32_t* bits = covbits + (size_t)i * kCovWords;
    bits[0] = w0; bits[1] = w1;
    if constexpr (kCovWords > 2) bits[kCovWords - 1] = w2;
    if (over || c0 > kCovBits) atomicOr(&ovf[i >> 5], 1u << (i & 31));   // the fill re-tests
    offc[i] = (uint16_t)(cnt - 1);   // minus the row's own atom
  }
  __syncthreads();
  // ---- degrees -> pose-local offsets, capacity check, row pointers ----
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    a.deg_cov[base + i] = offc[i];
    a.deg_ncov[base + i] = offn[i];
    if (!DIST) {   // scoring path: rows padded to 4 entries (see pad_rows)
      offc[i] = (offc[i] + 3) & ~3;
      offn[i] = (offn[i] + 3) & ~3;
    }
  }
  const int totc = block_scan_u16_to_global(offc, n, a.row_cov + base, cbase, warp_tot);
  const int totn = block_scan_u16_to_global(offn, n, a.row_ncov + base, cbase, warp_tot);
  if (totc > a.cap || totn > a.cap) {
    fail(FS_ERR_EDGE_CAP);
    return;
  }
  // pose-local row starts (written by the scans above)
  auto startc = [&](int i) { return (int)(a.row_cov[base + i] - cbase); };
  auto startn = [&](int i) { return (int)(a.row_ncov[base + i] - cbase); };

  // ---- fill non-covalent rows (ascending neighbour id) ----
  col_t* coln = a.col_ncov + cbase;
  double* distn = DIST ? a.dist_ncov + cbase : nullptr;
  if (use_mask) {
    for (int w = warp; w < W; w += kCsrWarps) {   // S rows 32w + lane: L ids ascending
      const int si = 32 * w + lane;
      const bool sv = si < nS;
      const int i = sv ? Slist[si] : 0;
      double xi, yi, zi; int32_t ei_, ri_;
      if (DIST && sv) pv.atom(i, xi, yi, zi, ei_, ri_);
      int o = sv ? startn(i) : 0;
      for (int l0 = 0; l0 < nL; l0 += 32) {
        // this chunk's mask words, transposed: lane l gets S atom 32w + l's
        // hits among L atoms l0 .. l0 + 31
        const int lj = l0 + lane;
        uint32_t bits = warp_transpose32(lj < nL ? mask[lj * W + w] : 0u, lane);
        while (bits) {
          const int b = __ffs(bits) - 1;
          bits &= bits - 1;
          const int j = Llist[l0 + b];
          FS_DCHECK(o < a.cap, "graph ncov S fill", o, a.cap);
          coln[o] = j;
          if (DIST) { double d; exact_edge(pv, xi, yi, zi, j, rmax2, a.tn, &d); distn[o] = d; }
          ++o;
        }
      }
    }
    for (int lj = threadIdx.x; lj < nL; lj += blockDim.x) {  // L rows: S ids ascending
      const int i = Llist[lj];
      int o = startn(i);
      double xi, yi, zi; int32_t ei_, ri_; pv.atom(i, xi, yi, zi, ei_, ri_);
      for (int w = 0; w < W; ++w) {
        uint32_t bits = mask[lj * W + w];
        while (bits) {
          const int b = __ffs(bits) - 1;
          bits &= bits - 1;
          const int j = Slist[32 * w + b];
          FS_DCHECK(o < a.cap, "graph ncov L fill", o, a.cap);
          coln[o] = j;
          if (DIST) { double d; exact_edge(pv, xi, yi, zi, j, rmax2, a.tn, &d); distn[o] = d; }
          ++o;
        }
      }
    }
  } else {
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
      double xi, yi, zi; int32_t ei_, ri_; pv.atom(i, xi, yi, zi, ei_, ri_);
      const float4 fi = pf[i];
      const int ri = (int)fi.w;
      const int ob = ri == 0 ? n0 : 0, oe = ri == 0 ? n : n0;
      int o = startn(i);
      for (int q = ob; q < oe; ++q) {
        const int j = role_list[q];
        const float4 fj = pf[j];
        const float dx = fi.x - fj.x, dy = fi.y - fj.y, dz = fi.z - fj.z;
        if (decide(dx * dx + dy * dy + dz * dz, n_lo2, n_hi2, xi, yi, zi, j, a.tn)) {
          coln[o] = j;
          if (DIST) { double d; exact_edge(pv, xi, yi, zi, j, rmax2, a.tn, &d); distn[o] = d; }
          ++o;
        }
      }
    }
  }
  if (!DIST) {
    const col_t padv = (col_t)((n + 15) & ~15);
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
      const int d = a.deg_ncov[base + i];
      for (int k = startn(i) + d; k & 3; ++k) coln[k] = padv;
    }
  }
  // ---- fill covalent rows.  Scoring path (no distances): rows stay in the
  // deterministic stencil order (cells x-, y-, z-major, ids ascending inside
  // a cell) -- a pose's sums never depend on its batch.  Featurizer path
  // (distances, edge lists compared bitwise with the reference): rows are
  // insertion-sorted to ascending neighbour id. ----
  col_t* colc = a.col_cov + cbase;
  double* distc = DIST ? a.dist_cov + cbase : nullptr;
  for (int idx = threadIdx.x; idx < n; idx += blockDim.x) {
    const int i = cell_list[idx];
    const int rb = startc(i);
    int o = rb;
    const uint32_t* bits = covbits + (size_t)i * kCovWords;
    if (!DIST && !((ovf[i >> 5] >> (i & 31)) & 1u)) {
      // replay the count pass's hits: candidate index c of a stencil column
      // run maps to cell_list[qb + c - c0]; the row's own atom (a candidate
      // that always hits) is not emitted
      // (a row that is not re-tested has < kCovBits candidates and <= 64 per
      // column: each column's hits are one 64-bit window of the kept bits)
      static_assert(kCovWords == 3, "covalent hit window assumes 96 kept bits");
      const int ri = (int)pf[i].w;
      const int kp = keys[i];
      const int cz = kp & 15, cy = (kp >> 4) & 15, cx = (kp >> 8) & 15;
      const uint64_t blo = (uint64_t)bits[0] | ((uint64_t)bits[1] << 32);
      const uint64_t bhi = bits[2];
      int c0 = 0;
      for (int dx = -1; dx <= 1; ++dx) {
        const int ax = cx + dx;
        if (ax < 0 || ax >= nca) continue;
        for (int dy = -1; dy <= 1; ++dy) {
          const int ay = cy + dy;
          if (ay < 0 || ay >= nca) continue;
          const int z0 = max(cz - 1, 0), z1 = min(cz + 1, nca - 1);
          const int k0 = ri * NC + (ax * nca + ay) * nca + z0, k1 = ri * NC + (ax * nca + ay) * nca + z1;
          const int qb = k0 == 0 ? 0 : cell_start[k0 - 1], qe = cell_start[k1];
          const int len = qe - qb;
          uint64_t cb = c0 >= 64 ? bhi >> (c0 - 64) : c0 == 0 ? blo : (blo >> c0) | (bhi << (64 - c0));
          if (len < 64) cb &= (1ull << len) - 1ull;
          while (cb) {
            const int b = __ffsll((long long)cb) - 1;
            cb &= cb - 1ull;
            const int j = cell_list[qb + b];
            FS_DCHECK(o < a.cap, "graph cov fill", o, a.cap);
            if (j != i) colc[o++] = (col_t)j;
          }
          c0 += len;
        }
      }
      continue;
    }
    cov_scan(i, [&](int j) {
      colc[o] = j;
      if (DIST) {
        double d;
        double xi, yi, zi; int32_t ei_, ri_; pv.atom(i, xi, yi, zi, ei_, ri_); exact_edge(pv, xi, yi, zi, j, rmax2, a.tc, &d);
        distc[o] = d;
      }
      ++o;
    });
    if constexpr (DIST) {   // featurizer path: ascending neighbour id
      for (int x = rb + 1; x < o; ++x) {
        const int v = colc[x];
        const double dv = distc[x];
        int y = x - 1;
        while (y >= rb && colc[y] > v) {
          colc[y + 1] = colc[y];
          distc[y + 1] = distc[y];
          --y;
        }
        colc[y + 1] = v;
        distc[y + 1] = dv;
      }
    }
  }
  if (!DIST) {
    // pad covalent rows to 4 entries with the all-zero node-state row (the
    // message-passing kernels read neighbour ids four at a time)
    const col_t padv = (col_t)((n + 15) & ~15);
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
      const int d = a.deg_cov[base + i];
      for (int k = startc(i) + d; k & 3; ++k) colc[k] = padv;
    }
  }
}

int launch_graph_csr(const fs_pose_batch& b, const int64_t* node_off, double tc, double tn, int64_t* row_cov,
                     int32_t* deg_cov, col_t* col_cov, double* dist_cov, int64_t* row_ncov, int32_t* deg_ncov,
                     col_t* col_ncov, double* dist_ncov, int64_t cap, int32_t* err, cudaStream_t st,
                     float* feats, int c_elem, double box) {
  if (!(tc >= 1.2 && tc <= 5.9) || !(tn >= 1.2 && tn <= 5.9)) return FS_EINVAL;   // complexes.py:228-231
  if (b.n_poses <= 0) return FS_OK;
  GraphCsrArgs a;
  a.feats = feats; a.c_elem = c_elem; a.box = box;
  a.b = b; a.node_off = node_off; a.tc = tc; a.tn = tn;
  a.row_cov = row_cov; a.deg_cov = deg_cov; a.col_cov = col_cov; a.dist_cov = dist_cov;
  a.row_ncov = row_ncov; a.deg_ncov = deg_ncov; a.col_ncov = col_ncov; a.dist_ncov = dist_ncov;
  // scoring path: pose slices start 4-aligned (rows are padded to 4 entries)
  a.cap = (dist_cov || dist_ncov) ? cap : (cap & ~static_cast<int64_t>(3)); a.err = err;
  int atoms = b.max_pose_atoms > 0 ? b.max_pose_atoms : FS_MAX_POSE_ATOMS;
  if (atoms > FS_MAX_POSE_ATOMS) atoms = FS_MAX_POSE_ATOMS;
  a.smem_atoms = atoms;
  const size_t smem = graph_csr_smem_bytes(atoms);
  if (dist_cov || dist_ncov) {
    FS_CUDA_CHECK(cudaFuncSetAttribute(graph_csr_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    graph_csr_kernel<true><<<b.n_poses, kCsrThreads, smem, st>>>(a);
  } else {
    FS_CUDA_CHECK(cudaFuncSetAttribute(graph_csr_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    graph_csr_kernel<false><<<b.n_poses, kCsrThreads, smem, st>>>(a);
  }
  FS_LAUNCH_CHECK();
  return FS_OK;
}


// ===========================================================================
// Pocket-factored radius graph (fs_score_poses_cached).
// A factorable pose is pocket atoms (all role 0) + ligand atoms (all role 1,
// at most kFactMaxLig).  Only edges that touch the ligand are built:
//   covalent     : ligand-ligand (pocket-pocket edges live in the cache)
//   non-covalent : ligand-pocket (bipartite, as in graph_csr_kernel)
// Compact node slice of pose p (rows p*S ..): ligand atoms [0, nL), zero rows
// up to nLp = roundup16(nL), then the nA pocket atoms with a ligand
// neighbour, ascending pocket id (aff[] = their pocket ids).  Neighbour order
// is ascending in the original node id, same predicate as the full kernel.
// ===========================================================================
struct GraphFactArgs {
  fs_pose_batch b;
  double tc, tn, box;
  int c_elem;
  int64_t S, cap;
  int32_t* cnt; int32_t* aff; float* feats;
  int64_t* row_cov; int32_t* deg_cov; col_t* col_cov;
  int64_t* row_ncov; int32_t* deg_ncov; col_t* col_ncov;
  int32_t* err;
  int max_pocket;
};

constexpr int kFactMaxLig = 128;
constexpr int kFactWords = kFactMaxLig / 32;

__host__ __device__ inline size_t graph_fact_smem_bytes(int max_pocket) {
  const size_t np4 = (size_t)((max_pocket + 3) & ~3), nc = np4 + kFactMaxLig + 32;
  return np4 * 16 + kFactMaxLig * 16 + np4 * kFactWords * 4 + (np4 + 4) * 4 + 2 * (nc + 4) * 4 + 256;
}

// thresholds are (-1, inf) when the prefilter is off: every pair is exact
__device__ __forceinline__ bool fact_decide(const PoseView& pv, float d2f, float lo2, float hi2, double xi, double yi,
                                            double zi, int j, double rmax2, double t) {
  if (d2f > hi2) return false;
  if (d2f <= lo2) return true;
  return exact_edge_slow(pv, xi, yi, zi, j, rmax2, t);
}

__global__ void __launch_bounds__(kCsrThreads) graph_fact_kernel(GraphFactArgs a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ int s_ncnt[kFactMaxLig];
  __shared__ int s_flag;
  __shared__ double s_red[kCsrWarps];
  __shared__ int warp_tot[32];
  const int p = blockIdx.x;
  const PoseView pv = pose_view(a.b, p);
  const int np = (int)pv.np_, nL = (int)pv.na;
  const int64_t nb = (int64_t)p * a.S, cb = (int64_t)p * a.cap;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  auto give_up = [&](int flags) {
    if (threadIdx.x == 0) { atomicOr(&a.err[p], flags); a.cnt[2 * p] = 0; a.cnt[2 * p + 1] = 0; }
  };
  if (np == 0 || np > a.max_pocket || nL > kFactMaxLig || np + nL > FS_MAX_POSE_ATOMS) {
    give_up(FS_ERR_NOT_FACTORED);
    return;
  }
  const int np4 = (a.max_pocket + 3) & ~3, ncmax = np4 + kFactMaxLig + 32;
  float4* pf = reinterpret_cast<float4*>(smem_raw);
  float4* lf = pf + np4;
  uint32_t* mask = reinterpret_cast<uint32_t*>(lf + kFactMaxLig);   // [np][kFactWords]
  int* rank = reinterpret_cast<int*>(mask + (size_t)np4 * kFactWords);   // [np + 1]
  int* offc = rank + np4 + 4;                                        // [nc + 1]
  int* offn = offc + ncmax + 4;
  if (threadIdx.x == 0) s_flag = 0;
  __syncthreads();

  // ---- atoms; the pose must be pocket(role 0) + ligand(role 1), finite ----
  double amax = 0.0;
  int bad = 0;
  for (int i = threadIdx.x; i < np + nL; i += blockDim.x) {
    double x, y, z; int32_t e, r;
    pv.atom(i, x, y, z, e, r);
    if (!isfinite(x) || !isfinite(y) || !isfinite(z) || r != (i < np ? 0 : 1)) bad = 1;
    amax = fmax(amax, fmax(fabs(x), fmax(fabs(y), fabs(z))));
    const float4 v = make_float4((float)x, (float)y, (float)z, 0.f);
    if (i < np) pf[i] = v; else lf[i - np] = v;
  }
  if (bad) atomicOr(&s_flag, 1);
  for (int o = 16; o > 0; o >>= 1) amax = fmax(amax, __shfl_xor_sync(0xffffffffu, amax, o));
  if (lane == 0) s_red[warp] = amax;
  __syncthreads();
  if (s_flag) { give_up(FS_ERR_NOT_FACTORED); return; }
  double absmax = 0.0;
  for (int w = 0; w < kCsrWarps; ++w) absmax = fmax(absmax, s_red[w]);
  const bool prefilter = absmax < 1024.0;
  const double rmax = fmax(a.tc, a.tn), rmax2 = __dmul_rn(rmax, rmax);
  const float delta = 1e-5f + 2e-6f * (float)absmax;
  const float c_lo2 = prefilter ? ((float)a.tc - delta) * ((float)a.tc - delta) : -1.0f;
  const float c_hi2 = prefilter ? ((float)a.tc + delta) * ((float)a.tc + delta) : INFINITY;
  const float n_lo2 = prefilter ? ((float)a.tn - delta) * ((float)a.tn - delta) : -1.0f;
  const float n_hi2 = prefilter ? ((float)a.tn + delta) * ((float)a.tn + delta) : INFINITY;
  const float n_mid2 = prefilter ? 0.5f * (n_lo2 + n_hi2) : 0.0f;
  const float n_half2 = prefilter ? 0.5f * (n_hi2 - n_lo2) * 1.0001f + 1e-6f : INFINITY;

  // ---- non-covalent (ligand x pocket) bitmasks: lanes over pocket atoms,
  // loop over the ligand atoms (broadcast reads); each lane builds its pocket
  // row's mask through ballots + warp transposes (no mask atomics),
  // ligand-row counts accumulate per lane; both fills read the masks. ----
  for (int i = threadIdx.x; i < kFactMaxLig; i += blockDim.x) s_ncnt[i] = 0;
  __syncthreads();
  {
    int acc[kFactWords] = {0, 0, 0, 0};   // lane l: hits of ligand atoms 32w + l
    const int nW = (nL + 31) / 32;
    for (int j0 = warp * 32; j0 < np; j0 += kCsrWarps * 32) {
      const int j = j0 + lane;
      const bool jv = j < np;
      // idle lanes sit at infinity: never a hit, never in the band
      const float4 fj = jv ? pf[j] : make_float4(INFINITY, INFINITY, INFINITY, 0.f);
      // lane l keeps the ballot of ligand atom 32w + l (fp32-certain hits);
      // warp transposes turn them into the pocket rows' masks; lanes that saw
      // the band (one distance to its middle, a superset) settle exactly
      uint32_t b[kFactWords] = {0u, 0u, 0u, 0u};
      float bmin = INFINITY;
#pragma unroll
      for (int w = 0; w < kFactWords; ++w) {
        const int s1 = min(nL, 32 * (w + 1));
#pragma unroll 4
        for (int s = 32 * w; s < s1; ++s) {
          const float4 fi = lf[s];
          const float dx = fi.x - fj.x, dy = fi.y - fj.y, dz = fi.z - fj.z;
          const float d2f = dx * dx + dy * dy + dz * dz;
          bmin = fminf(bmin, fabsf(d2f - n_mid2));
          const uint32_t bal = __ballot_sync(0xffffffffu, d2f <= n_lo2);
          b[w] = lane == s - 32 * w ? bal : b[w];
        }
      }
      uint32_t m[kFactWords] = {0u, 0u, 0u, 0u};
#pragma unroll
      for (int w = 0; w < kFactWords; ++w)
        if (w < nW) m[w] = warp_transpose32(b[w], lane);
      const bool band = bmin <= n_half2;
      if (__any_sync(0xffffffffu, band)) {   // rare: exact float64 predicate inside the band
        if (band) {
          for (int s = 0; s < nL; ++s) {
            const float4 fi = lf[s];
            const float dx = fi.x - fj.x, dy = fi.y - fj.y, dz = fi.z - fj.z;
            const float d2f = dx * dx + dy * dy + dz * dz;
            if (jv && d2f > n_lo2 && d2f <= n_hi2 && exact_pair_slow(pv, np + s, j, rmax2, a.tn)) {
#pragma unroll
              for (int w = 0; w < kFactWords; ++w)
                if (s >> 5 == w) m[w] |= 1u << (s & 31);
            }
          }
        }
#pragma unroll
        for (int w = 0; w < kFactWords; ++w)
          if (w < nW) b[w] = warp_transpose32(m[w], lane);
      }
#pragma unroll
      for (int w = 0; w < kFactWords; ++w) acc[w] += __popc(b[w]);
      if (jv) {
#pragma unroll
        for (int w = 0; w < kFactWords; ++w) mask[j * kFactWords + w] = m[w];
      }
    }
#pragma unroll
    for (int w = 0; w < kFactWords; ++w)
      if (acc[w]) atomicAdd(&s_ncnt[32 * w + lane], acc[w]);
  }
  // ligand-ligand covalent degrees: one warp per ligand atom
  for (int s = warp; s < nL; s += kCsrWarps) {
    double xi, yi, zi; int32_t e_, r_;
    pv.atom(np + s, xi, yi, zi, e_, r_);
    const float4 fi = lf[s];
    int cc = 0;
    for (int j0 = 0; j0 < nL; j0 += 32) {
      const int j = j0 + lane;
      bool hit = false;
      if (j < nL && j != s) {
        const float4 fj = lf[j];
        const float dx = fi.x - fj.x, dy = fi.y - fj.y, dz = fi.z - fj.z;
        hit = fact_decide(pv, dx * dx + dy * dy + dz * dz, c_lo2, c_hi2, xi, yi, zi, np + j, rmax2, a.tc);
      }
      cc += __popc(__ballot_sync(0xffffffffu, hit));
    }
    if (lane == 0) offc[s] = cc;
  }
  __syncthreads();
  for (int s = threadIdx.x; s < nL; s += blockDim.x) offn[s] = s_ncnt[s];
  for (int j = threadIdx.x; j < np; j += blockDim.x) {
    uint32_t any = 0u;
#pragma unroll
    for (int w = 0; w < kFactWords; ++w) any |= mask[j * kFactWords + w];
    rank[j] = any ? 1 : 0;
  }
  block_exclusive_scan(rank, np, warp_tot);
  const int nA = rank[np];
  const int nLp = (nL + 15) & ~15, nc = nLp + nA;
  if (nc > a.S) { give_up(FS_ERR_NOT_FACTORED); return; }
  for (int r = nL + threadIdx.x; r < nc; r += blockDim.x) { offc[r] = 0; if (r < nLp) offn[r] = 0; }
  for (int j = threadIdx.x; j < np; j += blockDim.x) {
    int c = 0;
#pragma unroll
    for (int w = 0; w < kFactWords; ++w) c += __popc(mask[j * kFactWords + w]);
    if (c) offn[nLp + rank[j]] = c;
  }
  __syncthreads();
  for (int r = threadIdx.x; r < nc; r += blockDim.x) {
    a.deg_cov[nb + r] = offc[r]; a.deg_ncov[nb + r] = offn[r];
    offc[r] = (offc[r] + 3) & ~3;   // rows padded to 4 entries (see the end)
    offn[r] = (offn[r] + 3) & ~3;
  }
  block_exclusive_scan(offc, nc, warp_tot);
  block_exclusive_scan(offn, nc, warp_tot);
  if (offc[nc] > a.cap || offn[nc] > a.cap) { give_up(FS_ERR_EDGE_CAP); return; }
  for (int r = threadIdx.x; r < nc; r += blockDim.x) { a.row_cov[nb + r] = cb + offc[r]; a.row_ncov[nb + r] = cb + offn[r]; }
  for (int j = threadIdx.x; j < np; j += blockDim.x) {
    uint32_t any = 0u;
#pragma unroll
    for (int w = 0; w < kFactWords; ++w) any |= mask[j * kFactWords + w];
    if (any) {
      FS_DCHECK(nLp + rank[j] < a.S, "aff", nLp + rank[j], a.S);
      a.aff[nb + nLp + rank[j]] = j;
    }
  }
  if (threadIdx.x == 0) { a.cnt[2 * p] = nL; a.cnt[2 * p + 1] = nA; }

  // ---- fill: ligand rows (covalent: ligand ids; non-covalent: compact pocket ids) ----
  col_t* colc = a.col_cov + cb;
  col_t* coln = a.col_ncov + cb;
  const unsigned below = (1u << lane) - 1u;
  for (int s = warp; s < nL; s += kCsrWarps) {
    double xi, yi, zi; int32_t e_, r_;
    pv.atom(np + s, xi, yi, zi, e_, r_);
    const float4 fi = lf[s];
    int o = offc[s];
    for (int j0 = 0; j0 < nL; j0 += 32) {
      const int j = j0 + lane;
      bool hit = false;
      if (j < nL && j != s) {
        const float4 fj = lf[j];
        const float dx = fi.x - fj.x, dy = fi.y - fj.y, dz = fi.z - fj.z;
        hit = fact_decide(pv, dx * dx + dy * dy + dz * dz, c_lo2, c_hi2, xi, yi, zi, np + j, rmax2, a.tc);
      }
      const unsigned m = __ballot_sync(0xffffffffu, hit);
      if (hit) {
        FS_DCHECK(o + __popc(m & below) < a.cap, "colc", o + __popc(m & below), a.cap);
        colc[o + __popc(m & below)] = j;
      }
      o += __popc(m);
    }
  }
  // ligand rows' pocket neighbours: warp w takes ligand atoms 32w + lane; each
  // 32-atom pocket chunk's mask words, transposed, are the lanes' hit bits
  for (int w = warp; w < (nL + 31) / 32; w += kCsrWarps) {
    const int s = 32 * w + lane;
    int o = s < nL ? offn[s] : 0;
    for (int j0 = 0; j0 < np; j0 += 32) {
      const int jl = j0 + lane;
      uint32_t bits = warp_transpose32(jl < np ? mask[jl * kFactWords + w] : 0u, lane);
      while (bits) {
        const int j = j0 + __ffs(bits) - 1;
        bits &= bits - 1;
        FS_DCHECK(o < a.cap, "coln lig", o, a.cap);
        FS_DCHECK(nLp + rank[j] < nc, "coln val", nLp + rank[j], nc);
        coln[o++] = nLp + rank[j];
      }
    }
  }
  // pocket rows: their ligand neighbours, ascending
  for (int j = threadIdx.x; j < np; j += blockDim.x) {
    int o = -1;
#pragma unroll
    for (int w = 0; w < kFactWords; ++w) {
      uint32_t bits = mask[j * kFactWords + w];
      if (bits && o < 0) o = offn[nLp + rank[j]];
      while (bits) {
        const int bt = __ffs(bits) - 1;
        bits &= bits - 1;
        FS_DCHECK(o >= 0 && o < a.cap, "coln pocket", o, a.cap);
        coln[o++] = 32 * w + bt;
      }
    }
  }
  // pad every row to 4 entries with the all-zero node-state row
  __syncthreads();
  {
    const col_t padv = (col_t)((nc + 15) & ~15);
    for (int r = threadIdx.x; r < nc; r += blockDim.x) {
      for (int k = offc[r] + a.deg_cov[nb + r]; k & 3; ++k) colc[k] = padv;
      for (int k = offn[r] + a.deg_ncov[nb + r]; k & 3; ++k) coln[k] = padv;
    }
  }
  // ligand node features, as node_features_kernel<float> (complexes.py:233-236)
  const int F = a.c_elem + 4;
  for (int s = threadIdx.x; s < nL; s += blockDim.x) {
    double x, y, z; int32_t e, r;
    pv.atom(np + s, x, y, z, e, r);
    float* f = a.feats + (nb + s) * F;
    const int ec = min(max(e, 0), a.c_elem - 1);
    for (int c = 0; c < a.c_elem; ++c) f[c] = c == ec ? 1.f : 0.f;
    f[a.c_elem] = (float)r;
    f[a.c_elem + 1] = (float)__dadd_rn(__ddiv_rn(x, a.box), 0.5);
    f[a.c_elem + 2] = (float)__dadd_rn(__ddiv_rn(y, a.box), 0.5);
    f[a.c_elem + 3] = (float)__dadd_rn(__ddiv_rn(z, a.box), 0.5);
  }
}

int launch_graph_fact(const fs_pose_batch& b, double tc, double tn, double box, int c_elem, int64_t S, int64_t cap,
                      int max_pocket, int32_t* cnt, int32_t* aff, float* feats, int64_t* row_cov, int32_t* deg_cov,
                      col_t* col_cov, int64_t* row_ncov, int32_t* deg_ncov, col_t* col_ncov, int32_t* err,
                      cudaStream_t st) {
  if (!(tc >= 1.2 && tc <= 5.9) || !(tn >= 1.2 && tn <= 5.9)) return FS_EINVAL;
  if (b.n_poses <= 0) return FS_OK;
  GraphFactArgs a;
  a.b = b; a.tc = tc; a.tn = tn; a.box = box; a.c_elem = c_elem; a.S = S; a.cap = cap & ~static_cast<int64_t>(3);
  a.cnt = cnt; a.aff = aff; a.feats = feats;
  a.row_cov = row_cov; a.deg_cov = deg_cov; a.col_cov = col_cov;
  a.row_ncov = row_ncov; a.deg_ncov = deg_ncov; a.col_ncov = col_ncov;
  a.err = err; a.max_pocket = max_pocket;
  const size_t smem = graph_fact_smem_bytes(max_pocket);
  if (smem > 227 * 1024) return FS_ECAPACITY;
  FS_CUDA_CHECK(cudaFuncSetAttribute(graph_fact_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  graph_fact_kernel<<<b.n_poses, kCsrThreads, smem, st>>>(a);
  FS_LAUNCH_CHECK();
  return FS_OK;
}

// ===========================================================================
// Inspection of the scoring-path graphs (fs_scoring_graph): every DIRECTED
// CSR entry (i, j) that graph_csr_kernel / graph_fact_kernel left for the
// SG-CNN, mapped back to the pose's original node numbering (pocket atoms,
// then its own atoms), with the float64 distance of the pair recomputed by
// the reference's formula (the scoring kernels never store distances).
// Padding entries (rows are padded to 4 ids) are not listed.
// ===========================================================================
struct CsrEntriesArgs {
  fs_pose_batch b;
  const int64_t* node_off;                          // full mode
  const int32_t* fact_cnt; const int32_t* aff;      // factored mode (null: full)
  int64_t S, cap, cap_out;
  const int64_t* row[2]; const int32_t* deg[2]; const col_t* col[2];
  int32_t* n_out[2]; int32_t* ent[2]; double* dist[2];
  const int32_t* err;
};

__global__ void __launch_bounds__(256) csr_entries_kernel(CsrEntriesArgs a) {
  extern __shared__ int s_off[];      // [rows + 1]
  __shared__ int warp_tot[32];
  const int p = blockIdx.x;
  const PoseView pv = pose_view(a.b, p);
  const bool fact = a.fact_cnt != nullptr;
  const int np = (int)pv.np_;
  int rows, nL = 0, nLp = 0;
  int64_t nb;
  if (fact) {
    nL = a.fact_cnt[2 * p];
    nLp = (nL + 15) & ~15;
    rows = nLp + a.fact_cnt[2 * p + 1];
    nb = (int64_t)p * a.S;
  } else {
    nb = a.node_off[p];
    rows = (int)(a.node_off[p + 1] - nb);
  }
  if (a.err[p]) {
    if (threadIdx.x < 2) a.n_out[threadIdx.x][p] = 0;
    return;
  }
  // compact factored row -> original node id (ligand rows, zero pad rows, touched pocket atoms)
  auto node_id = [&](int r) -> int {
    if (!fact) return r;
    return r < nL ? np + r : (r >= nLp ? a.aff[nb + r] : -1);
  };
  for (int t = 0; t < 2; ++t) {
    for (int r = threadIdx.x; r < rows; r += blockDim.x) s_off[r] = a.deg[t][nb + r];
    block_exclusive_scan(s_off, rows, warp_tot);
    const int64_t cb = (int64_t)p * a.cap, ob = (int64_t)p * a.cap_out;
    const int total = s_off[rows];
    for (int r = threadIdx.x; r < rows; r += blockDim.x) {
      const int d = a.deg[t][nb + r];
      if (!d) continue;
      const int i = node_id(r);
      double xi, yi, zi; int32_t e_, r_;
      pv.atom(i, xi, yi, zi, e_, r_);
      const int64_t s = a.row[t][nb + r] - cb;
      for (int k = 0; k < d; ++k) {
        const int j = node_id(a.col[t][cb + s + k]);
        const int64_t o = ob + s_off[r] + k;
        if (s_off[r] + k >= a.cap_out) break;
        a.ent[t][2 * o] = i;
        a.ent[t][2 * o + 1] = j;
        if (a.dist[t]) {
          double xj, yj, zj;
          pv.atom(j, xj, yj, zj, e_, r_);
          a.dist[t][o] = __dsqrt_rn(dist2_exact(xi - xj, yi - yj, zi - zj));
        }
      }
    }
    if (threadIdx.x == 0) a.n_out[t][p] = total;
    __syncthreads();
  }
}

int launch_csr_entries(const fs_pose_batch& b, const int64_t* node_off, const int32_t* fact_cnt, const int32_t* aff,
                       int64_t S, int64_t cap, int max_rows, const int64_t* row_cov, const int32_t* deg_cov,
                       const col_t* col_cov, const int64_t* row_ncov, const int32_t* deg_ncov, const col_t* col_ncov,
                       int64_t cap_out, int32_t* n_cov, int32_t* n_ncov, int32_t* ent_cov, int32_t* ent_ncov,
                       double* d_cov, double* d_ncov, const int32_t* err, cudaStream_t st) {
  if (b.n_poses <= 0) return FS_OK;
  CsrEntriesArgs a;
  a.b = b; a.node_off = node_off; a.fact_cnt = fact_cnt; a.aff = aff; a.S = S;
  // the scoring kernels round their slice capacity down to 4 entries
  a.cap = cap & ~static_cast<int64_t>(3); a.cap_out = cap_out;
  a.row[0] = row_cov; a.row[1] = row_ncov; a.deg[0] = deg_cov; a.deg[1] = deg_ncov;
  a.col[0] = col_cov; a.col[1] = col_ncov; a.n_out[0] = n_cov; a.n_out[1] = n_ncov;
  a.ent[0] = ent_cov; a.ent[1] = ent_ncov; a.dist[0] = d_cov; a.dist[1] = d_ncov; a.err = err;
  const size_t smem = (size_t)(max_rows + 2) * 4;
  FS_CUDA_CHECK(cudaFuncSetAttribute(csr_entries_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  csr_entries_kernel<<<b.n_poses, 256, smem, st>>>(a);
  FS_LAUNCH_CHECK();
  return FS_OK;
}

}  // namespace fs
