// SG-CNN head on the tensor cores (mma.sync m16n8k16 bf16, fp32 accumulate)
// for the reference widths (gather_width_cov 24, gather_width_noncov 128).
//
// Same math as gnn.cu (models.py:334-371): per step
//   [z|r] = sigma([s|h] . [[Wmsg.Wz  Wmsg.Wr]; [Uz Ur]] + [bz|br])
//   hh    = tanh ([s|r*h] . [[Wmsg.Wh]; [Uh]] + bh);   h <- h + z*(hh-h)
// with s = sum of neighbour h rows.  Each step walks 16-node tiles (rows
// counting-sorted by degree): (1) S = the tile's neighbour sums -- on the
// fp16 path (VAR & 16) as identity-A MMAs over ldmatrix.trans-loaded
// neighbour rows (see "tensor-core neighbour sums"), on the 3-pass path as
// per-lane fp32 gathers with whole-warp heavy rows (kHeavyDeg); (2) the GRU
// update of the tile on the tensor cores.
// The m16n8k16 fragment layouts line up so that each lane holds, for rows
// g and g+8 (g = lane/4), exactly the columns {2t,2t+1,8+2t,9+2t,16+2t,17+2t}
// (t = lane%4) of s, h, z, r, hh and h': the whole GRU update is lane-local
// and r*h feeds the second GEMM without any data exchange.
// SPLIT = 3 keeps fp32-class accuracy: x = hi + lo (bf16 each) and
// A.B ~ Ahi.Bhi + Ahi.Blo + Alo.Bhi (relative error ~2^-16); SPLIT = 2 splits
// the activations into fp16 hi + lo (22 significant bits) against fp16
// weights (2^-12 relative rounding): two passes, half the weight-fragment
// shared-memory traffic of SPLIT = 3; SPLIT = 1 is a
// single bf16 pass.  Node states stay fp32 in shared memory (the fp16 path
// gathers from double-buffered fp16 copies).
// Determinism: every row's sum has a fixed order that depends on its own CSR
// list only (CSR order; even / odd chunk accumulators on the MMA path; for
// heavy rows 8 CSR-strided partial sums in a fixed tree), a row's GEMM
// precision choice is a function of the row alone, fixed reduction trees,
// fixed pool order -> a pose's latent is bitwise independent of its batch.
#include <cstdlib>
#include <type_traits>

#include <cuda_fp16.h>

#include "common.cuh"
#include "gnn_mma.cuh"

namespace fs {


constexpr int kMaxMmaWarps = 24;   // smem reduction buffers are sized for this many warps
constexpr int kZrWords = 3 * 6 * 64;      // [kt][nt][lane][2] per hi/lo
constexpr int kHhWords = 3 * 3 * 64;
constexpr int kPhaseWords = 2 * (kZrWords + kHhWords);   // hi and lo
constexpr int kGatherWords = 2 * 2 * 32 * 64;

int gnn_mma_phase_words() { return kPhaseWords; }

#ifdef FS_GNN_PROF
// per-warp clock64 timeline of the first 8 poses (profiling builds only):
// [pose][slot][warp][4]; slot 0: (kernel start, embedding done), slots 1..9:
// steps (loop start, loop end, items, gather cycles, claim cycles, GRU
// cycles), slot 10: (pool done)
__device__ unsigned long long fs_gnn_prof_buf[8][12][kMaxMmaWarps][7];
#define GPROF(slot, k, v) do { if (blockIdx.x < 8) fs_gnn_prof_buf[blockIdx.x][slot][warp][k] = (v); } while (0)
#else
#define GPROF(slot, k, v) do {} while (0)
#endif
int gnn_mma_gather_words() { return kGatherWords; }

__device__ __forceinline__ void mma_bf16(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

__device__ __forceinline__ void mma_bf16_k8(float (&d)[4], uint32_t a0, uint32_t a1, uint32_t b0) {
  asm volatile(
      "mma.sync.aligned.m16n8k8.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a0), "r"(a1), "r"(b0));
}

template <int SPLIT>
__device__ __forceinline__ void mma_t(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  if constexpr (SPLIT == 2) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%0,%1,%2,%3};"
        : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
  } else {
    mma_bf16(d, a, b0, b1);
  }
}
template <int SPLIT>
__device__ __forceinline__ void mma_t_k8(float (&d)[4], uint32_t a0, uint32_t a1, uint32_t b0) {
  if constexpr (SPLIT == 2) {
    asm volatile("mma.sync.aligned.m16n8k8.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};"
                 : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
                 : "r"(a0), "r"(a1), "r"(b0));
  } else {
    mma_bf16_k8(d, a0, a1, b0);
  }
}

__device__ __forceinline__ uint32_t pack_bf16(float lo_idx, float hi_idx) {
  __nv_bfloat162 v = __floats2bfloat162_rn(lo_idx, hi_idx);
  return *reinterpret_cast<uint32_t*>(&v);
}
// split a pair into (hi, lo) bf16x2 words
__device__ __forceinline__ void fadd2(float& a0, float& a1, float b0, float b1);
__device__ __forceinline__ void split2(float x0, float x1, uint32_t& hi, uint32_t& lo) {
  __nv_bfloat162 h = __floats2bfloat162_rn(x0, x1);
  float2 hf = __bfloat1622float2(h);
  fadd2(x0, x1, -hf.x, -hf.y);   // exact: x - bf16(x)
  __nv_bfloat162 l = __floats2bfloat162_rn(x0, x1);
  hi = *reinterpret_cast<uint32_t*>(&h);
  lo = *reinterpret_cast<uint32_t*>(&l);
}

// A fragments of a 16x48 tile [left(24) | right(24)] from the lane's values:
// L[r][c] / R[r][c]: r in {row g, row g+8}, c in {2t,2t+1,8+2t,9+2t,16+2t,17+2t}
// fp16 hi/lo of a pair: lo = x - fp16(x) rounded to fp16
__device__ __forceinline__ void split2_f16(float x0, float x1, uint32_t& hi, uint32_t& lo) {
  __half2 h = __floats2half2_rn(x0, x1);
  float2 hf = __half22float2(h);
  fadd2(x0, x1, -hf.x, -hf.y);
  __half2 l = __floats2half2_rn(x0, x1);
  hi = *reinterpret_cast<uint32_t*>(&h);
  lo = *reinterpret_cast<uint32_t*>(&l);
}

template <int SPLIT>
__device__ __forceinline__ void put_a(uint32_t (&hi)[4], uint32_t (&lo)[4], int q, float x0, float x1) {
  if (SPLIT == 3) split2(x0, x1, hi[q], lo[q]);
  else if (SPLIT == 2) split2_f16(x0, x1, hi[q], lo[q]);
  else if (SPLIT == 5) { const __half2 v = __floats2half2_rn(x0, x1); hi[q] = *reinterpret_cast<const uint32_t*>(&v); }
  else hi[q] = pack_bf16(x0, x1);
}

// A fragments of a 16x48 tile [left(24) | right(24)] from the lane's values
// L[r][c], R[r][c] (r: rows g, g+8; c indexes cols 2t,2t+1,8+2t,9+2t,16+2t,17+2t):
// k-tile 0 = L[0..15]; k-tile 1 = L[16..23] | R[0..7]; k-tile 2 = R[8..23].
template <int SPLIT>
__device__ __forceinline__ void build_a48(const float (&L)[2][6], const float (&R)[2][6], uint32_t (&hi)[3][4],
                                          uint32_t (&lo)[3][4]) {
  put_a<SPLIT>(hi[0], lo[0], 0, L[0][0], L[0][1]);
  put_a<SPLIT>(hi[0], lo[0], 1, L[1][0], L[1][1]);
  put_a<SPLIT>(hi[0], lo[0], 2, L[0][2], L[0][3]);
  put_a<SPLIT>(hi[0], lo[0], 3, L[1][2], L[1][3]);
  put_a<SPLIT>(hi[1], lo[1], 0, L[0][4], L[0][5]);
  put_a<SPLIT>(hi[1], lo[1], 1, L[1][4], L[1][5]);
  put_a<SPLIT>(hi[1], lo[1], 2, R[0][0], R[0][1]);
  put_a<SPLIT>(hi[1], lo[1], 3, R[1][0], R[1][1]);
  put_a<SPLIT>(hi[2], lo[2], 0, R[0][2], R[0][3]);
  put_a<SPLIT>(hi[2], lo[2], 1, R[1][2], R[1][3]);
  put_a<SPLIT>(hi[2], lo[2], 2, R[0][4], R[0][5]);
  put_a<SPLIT>(hi[2], lo[2], 3, R[1][4], R[1][5]);
}

__device__ __forceinline__ void mma_bf16_c(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1,
                                           const float (&c)[4]) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%10,%11,%12,%13};"
      : "=f"(d[0]), "=f"(d[1]), "=f"(d[2]), "=f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1), "f"(c[0]), "f"(c[1]), "f"(c[2]),
        "f"(c[3]));
}

__device__ __forceinline__ void mma_f16_c(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1,
                                          const float (&c)[4]) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%10,%11,%12,%13};"
      : "=f"(d[0]), "=f"(d[1]), "=f"(d[2]), "=f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1), "f"(c[0]), "f"(c[1]), "f"(c[2]),
        "f"(c[3]));
}

// KT0 = 1: k-tile 0 (neighbour sums s[0..15]) is all zero and skipped (the
// products it would add are exact zeros)
// LO0 = false: k-tile 0 has no lo term (its A is a single fp16 pass)
// D = C + A.B, C = the gate biases of columns 8nt+2t, 8nt+2t+1 (both rows),
// entering as the C operand of each chain's first MMA.  LOM (SPLIT 2): the
// k-tiles that carry a lo pass (bit kt); SPLIT 3 always takes all three terms.
template <int SPLIT>
__device__ __forceinline__ void mma_c2(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1, float c0,
                                       float c1) {
  if constexpr (SPLIT == 2) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%10,%11,%10,%11};"
        : "=f"(d[0]), "=f"(d[1]), "=f"(d[2]), "=f"(d[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1), "f"(c0), "f"(c1));
  } else {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%10,%11,%10,%11};"
        : "=f"(d[0]), "=f"(d[1]), "=f"(d[2]), "=f"(d[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1), "f"(c0), "f"(c1));
  }
}
template <int SPLIT, int NT, int KT0 = 0, int LOM = 7>
__device__ __forceinline__ void gemm48(float (&D)[NT][4], const float (&C)[NT][2], const uint32_t (&ahi)[3][4],
                                       const uint32_t (&alo)[3][4], const uint32_t* __restrict__ fhi,
                                       const uint32_t* __restrict__ flo, int lane) {
  // small cross terms first, the hi.hi product last, all into one
  // accumulator: NT independent chains keep the tensor pipe busy
#pragma unroll
  for (int kt = KT0; kt < 3; ++kt)
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) {
      const uint2 bh = *reinterpret_cast<const uint2*>(fhi + ((kt * NT + nt) * 32 + lane) * 2);
      bool first = kt == KT0;
      if constexpr (SPLIT == 3) {
        const uint2 bl = *reinterpret_cast<const uint2*>(flo + ((kt * NT + nt) * 32 + lane) * 2);
        if (first) mma_c2<3>(D[nt], alo[kt], bh.x, bh.y, C[nt][0], C[nt][1]);
        else mma_bf16(D[nt], alo[kt], bh.x, bh.y);
        mma_bf16(D[nt], ahi[kt], bl.x, bl.y);
        first = false;
      } else if constexpr (SPLIT == 2) {
        if ((LOM >> kt) & 1) {
          if (first) mma_c2<2>(D[nt], alo[kt], bh.x, bh.y, C[nt][0], C[nt][1]);
          else mma_t<2>(D[nt], alo[kt], bh.x, bh.y);
          first = false;
        }
      }
      if (first) mma_c2<SPLIT>(D[nt], ahi[kt], bh.x, bh.y, C[nt][0], C[nt][1]);
      else mma_t<SPLIT>(D[nt], ahi[kt], bh.x, bh.y);
    }
}

// Rows with at least kHeavyDeg neighbours are summed by a whole warp (8
// neighbours per iteration, fixed-tree combine); lighter rows are summed 16
// at a time in degree-sorted tiles, so a tile's lanes run out of neighbours
// together.  Both forms read 8 (row, neighbour) pairs per 12 lane-instructions.
constexpr int kHeavyDeg = 32;
constexpr int kBins = kHeavyDeg + 1;
// tensor-core gathers (VAR & 16) have no heavy rows: a finer degree sort
// (degrees 0..kNatBins-2, the rest in one bin) keeps tile padding low
// (NAT: hist + cursors live in the unused heavy-sum buffer)
constexpr int kNatBins = 129;
#ifndef FS_POOL_SPLIT
#define FS_POOL_SPLIT 4
#endif
constexpr int kPoolSplit = FS_POOL_SPLIT;   // pool items per 16-row tile (column groups split evenly)
// VAR & 32: a row's neighbour sums take one fp16 pass (its lo term zeroed)
// while all its |s| <= kSBig: rounding <= kSBig * 2^-12 absolute, the order
// of the fp16-rounded rows they sum; larger sums keep the hi/lo split.
// Measured: config-1 max rel. 7.6e-4 vs the oracle; the dense stress pocket
// (sums of ~600 rows) within 3e-3.
#ifndef FS_SBIG
#define FS_SBIG 16.0f
#endif
constexpr float kSBig = FS_SBIG;
constexpr int kCtlWords = 6 + 2 * kBins;

// ---- tensor-core neighbour sums (VAR & 16) --------------------------------
// S(16 rows x 24) += I16 . B, B = the c-th neighbour row of each of the tile's
// 16 rows (fp16 gather copies, natural column order, 48-byte rows), loaded
// k-major by ldmatrix.trans straight into m16n8k16 B fragments; the identity
// A makes the tensor core an fp32 adder (one nonzero product per output), and
// the D fragments are the A-fragment layout of the GRU GEMM.
__device__ __forceinline__ void ldsm_x4_t(uint32_t (&r)[4], uint32_t addr) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(addr));
}
__device__ __forceinline__ void mma_f16_id(float (&d)[4], uint32_t ai, uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%5,%4}, {%6,%7}, "
      "{%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(ai), "r"(0u), "r"(b0), "r"(b1));
}
// the same with C = 0 (a chain's first chunk: no accumulator zeroing)
__device__ __forceinline__ void mma_f16_id0(float (&d)[4], uint32_t ai, uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%5,%4}, {%6,%7}, "
      "{%8,%8,%8,%8};"
      : "=f"(d[0]), "=f"(d[1]), "=f"(d[2]), "=f"(d[3])
      : "r"(ai), "r"(0u), "r"(b0), "r"(b1), "f"(0.0f));
}

// Node-state rows are stored lane-major: the 6 columns lane t owns in the
// MMA fragments ({2t,2t+1, 8+2t,9+2t, 16+2t,17+2t}) sit contiguously at
// 6t..6t+5, so a gathered row is two loads per lane (one 16-byte, one
// 8-byte) instead of three 8-byte ones, with fewer bank conflicts.  The
// 16-byte half is at 6t (t even) or 6t+2 (t odd); sums are kept in that
// storage order and mapped to fragment order once per row.
// packed fp32 add (sm_100 FADD2): two IEEE round-to-nearest adds, bitwise
// the same as two FADDs, one issue slot
__device__ __forceinline__ void fadd2(float& a0, float& a1, float b0, float b1) {
  asm("{\n.reg .b64 ra, rb;\n"
      "mov.b64 ra, {%0, %1};\n"
      "mov.b64 rb, {%2, %3};\n"
      "add.rn.f32x2 ra, ra, rb;\n"
      "mov.b64 {%0, %1}, ra;\n}"
      : "+f"(a0), "+f"(a1)
      : "f"(b0), "f"(b1));
}
__device__ __forceinline__ void fmul2(float& a0, float& a1, float b0, float b1) {
  asm("{\n.reg .b64 ra, rb;\n"
      "mov.b64 ra, {%0, %1};\n"
      "mov.b64 rb, {%2, %3};\n"
      "mul.rn.f32x2 ra, ra, rb;\n"
      "mov.b64 {%0, %1}, ra;\n}"
      : "+f"(a0), "+f"(a1)
      : "f"(b0), "f"(b1));
}
// a = a * b + c
__device__ __forceinline__ void ffma2(float& a0, float& a1, float b0, float b1, float c0, float c1) {
  asm("{\n.reg .b64 ra, rb, rc;\n"
      "mov.b64 ra, {%0, %1};\n"
      "mov.b64 rb, {%2, %3};\n"
      "mov.b64 rc, {%4, %5};\n"
      "fma.rn.f32x2 ra, ra, rb, rc;\n"
      "mov.b64 {%0, %1}, ra;\n}"
      : "+f"(a0), "+f"(a1)
      : "f"(b0), "f"(b1), "f"(c0), "f"(c1));
}
// (sigmoid, sigmoid) / (tanh, tanh) of a pre-scaled pair (see fs_sigmoid_pre)
__device__ __forceinline__ void sigmoid_pre2(float& u0, float& u1) {
  u0 = fs_ex2(u0); u1 = fs_ex2(u1);
  fadd2(u0, u1, 1.0f, 1.0f);
  u0 = fs_rcp(u0); u1 = fs_rcp(u1);
}
__device__ __forceinline__ void tanh_pre2(float& u0, float& u1) {
  sigmoid_pre2(u0, u1);
  ffma2(u0, u1, -2.0f, -2.0f, 1.0f, 1.0f);
}
// accumulate neighbour row j from the lane's two per-step bases (H4 = H + 6t
// + 2(t&1): its 16-byte half, H2: its 8-byte half): one multiply-add each
__device__ __forceinline__ void acc_row_at(float (&q)[4], float (&d)[2], const float* __restrict__ H4,
                                           const float* __restrict__ H2, int j) {
  const float4 v = *reinterpret_cast<const float4*>(H4 + j * 24);
  const float2 w = *reinterpret_cast<const float2*>(H2 + j * 24);
  fadd2(q[0], q[1], v.x, v.y);
  fadd2(q[2], q[3], v.z, v.w);
  fadd2(d[0], d[1], w.x, w.y);
}
// fp16 gather copies (VAR & 4): the same lane-major storage order, 48-byte
// rows; the lane's 16-byte fp32 half is an 8-byte fp16 load at half index
// 6t + 2(t&1), its 8-byte half a 4-byte load at 6t + (t&1 ? 0 : 4).  Mixed
// precision FHADD (fp32 += fp16, exact conversion): the sums stay fp32 and
// exactly CSR-ordered.
__device__ __forceinline__ void fhadd2(float& a0, float& a1, uint32_t v) {
  asm("{\n.reg .f16 l, h;\n"
      "mov.b32 {l, h}, %2;\n"
      "add.rn.f32.f16 %0, l, %0;\n"
      "add.rn.f32.f16 %1, h, %1;\n}"
      : "+f"(a0), "+f"(a1)
      : "r"(v));
}
__device__ __forceinline__ void acc_row_at16(float (&q)[4], float (&d)[2], const __half* __restrict__ G4,
                                             const __half* __restrict__ G2, int j) {
  const uint2 v = *reinterpret_cast<const uint2*>(G4 + j * 24);
  const uint32_t w = *reinterpret_cast<const uint32_t*>(G2 + j * 24);
  fhadd2(q[0], q[1], v.x);
  fhadd2(q[2], q[3], v.y);
  fhadd2(d[0], d[1], w);
}
// gate activations of a pair.  VAR & 3 (the fp16 2-pass path): the fp16
// weights are tanh-scaled (z, r by 1/2: sigmoid(x) = (1 + tanh(x/2)) / 2;
// h~ by 1), VAR & 1: one tanh.approx.f32 per value, VAR & 2: one
// tanh.approx.f16x2 per pair.  Else the ex2-scaled bf16 weights (see
// fs_sigmoid_pre / fs_tanh_pre): ex2 + rcp per value.
template <int VAR>
__device__ __forceinline__ void gate_tanh2(float& u0, float& u1) {
  if constexpr (VAR & 2) {
    const __half2 x = __floats2half2_rn(u0, u1);
    uint32_t xi = *reinterpret_cast<const uint32_t*>(&x), yi;
    asm("tanh.approx.f16x2 %0, %1;" : "=r"(yi) : "r"(xi));
    const float2 y = __half22float2(*reinterpret_cast<const __half2*>(&yi));
    u0 = y.x; u1 = y.y;
  } else {
    asm("tanh.approx.f32 %0, %1;" : "=f"(u0) : "f"(u0));
    asm("tanh.approx.f32 %0, %1;" : "=f"(u1) : "f"(u1));
  }
}
template <int VAR>
__device__ __forceinline__ void gate_sigmoid2(float& u0, float& u1) {
  if constexpr ((VAR & 3) != 0) {
    gate_tanh2<VAR>(u0, u1);
    ffma2(u0, u1, 0.5f, 0.5f, 0.5f, 0.5f);
  } else {
    sigmoid_pre2(u0, u1);
  }
}
template <int VAR>
__device__ __forceinline__ void gate_tanh_pre2(float& u0, float& u1) {
  if constexpr ((VAR & 3) != 0) gate_tanh2<VAR>(u0, u1);
  else tanh_pre2(u0, u1);
}

__device__ __forceinline__ void frag_order(const float (&q)[4], const float (&d)[2], int t, float (&o)[6]) {
  const bool odd = t & 1;
  o[0] = odd ? d[0] : q[0]; o[1] = odd ? d[1] : q[1];
  o[2] = odd ? q[0] : q[2]; o[3] = odd ? q[1] : q[3];
  o[4] = odd ? q[2] : d[0]; o[5] = odd ? q[3] : d[1];
}
// storage position of natural column c (c = 8k + 2t + e -> 6t + 2k + e)
__host__ __device__ constexpr int hpos(int c) { return 6 * ((c % 8) / 2) + 2 * (c / 8) + (c % 2); }

// VAR (SPLIT 2 only): bit 0/1 = gate activations (see gate_tanh2); bit 2 =
// neighbour gathers from fp16 copies of the node states (the fp32 states are
// then single-buffered and updated in place: a row's fp32 state is read only
// by the warp that updates it)
template <int SPLIT, bool FACT, int kMmaWarps, int VAR = 0>
__global__ void __launch_bounds__(kMmaWarps * 32, 1) gnn_mma_kernel(GnnMmaArgs a) {
  constexpr bool G16 = (VAR & 4) != 0;
  constexpr bool NAT = (VAR & 16) != 0;   // tensor-core gathers, natural-order fp16 copies
  static_assert(!NAT || (G16 && SPLIT == 2), "tensor-core gathers read the fp16 copies");
  static_assert(SPLIT != 2 || (VAR & 3) != 0, "the fp16 weights are tanh-scaled");
  constexpr int NB = NAT ? kNatBins : kBins;   // degree bins of the gather-order sort
  extern __shared__ __align__(16) float sm[];
  __shared__ int wcnt[kMmaWarps];
  const int p = blockIdx.x;
  int64_t base;
  int n, nL = 0, nLp = 0;
  const char* pc = nullptr;   // this pose's pocket cache
  if constexpr (FACT) {
    base = static_cast<int64_t>(p) * a.fact_stride;
    nL = a.fact_cnt[2 * p];
    nLp = (nL + 15) & ~15;
    n = nLp + a.fact_cnt[2 * p + 1];
    pc = a.cache + static_cast<int64_t>(a.pose_target[p]) * a.cache_stride;
  } else {
    base = a.node_off[p];
    n = static_cast<int>(a.node_off[p + 1] - base);
  }
  // rows that hold a node (factored slices have zero rows between ligand and pocket)
  auto valid = [&](int r) { return FACT ? (r < nL || (r >= nLp && r < n)) : r < n; };
  float* lat = a.lat + static_cast<int64_t>(p) * a.ld_lat;
  if (a.err && a.err[p]) {
    for (int k = threadIdx.x; k < 128; k += blockDim.x) lat[k] = __int_as_float(0x7fc00000);
    return;
  }
  const int ntiles = (n + 15) / 16, npad = ntiles * 16;
  const int hrows = max(npad + 1, kMaxMmaWarps * 16);   // Hn doubles as the pool's reduction buffers
  // Hc / Hn: node states [npad + 1][24], double buffered (row npad stays zero:
  // padded gathers read it).  HS: neighbour sums of the heavy rows.
  float* Hc = sm;
  float* Hn = Hc + hrows * 24;      // both buffers hrows: either may end as Hn
  float* HS = Hn + hrows * 24;
  // G16: Hc = the fp32 states (never swapped); the Hn region holds the two
  // fp16 gather copies [hrows][24] each
  __half* Gc = reinterpret_cast<__half*>(Hn);
  __half* Gn = Gc + hrows * 24;
  uint32_t* WF = reinterpret_cast<uint32_t*>(HS + a.heavy_cap * 24);   // phase fragments
  float* WB = reinterpret_cast<float*>(WF + kPhaseWords);            // phase biases [72]
  int* CTL = reinterpret_cast<int*>(WB + 72);    // item ctr[2], heavy-done ctr[2], -, -, hist[kBins], cursor[kBins]
  int* hist = CTL + 6;
  uint16_t* PERM = reinterpret_cast<uint16_t*>(CTL + kCtlWords);   // gather order [npad]
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;
  GPROF(0, 0, clock64());
#define COLS(c) ((c) < 2 ? 2 * t + (c) : (c) < 4 ? 6 + 2 * t + (c) : 12 + 2 * t + (c))
#define PCOL(c) (6 * t + (c))   // storage position of the lane's c-th state column
  // NAT: both fp16 gather copies of a row from its 24 states in storage order
  auto store_nat16 = [&](__half* d0, __half* d1, const float (&hv)[24]) {
    uint32_t w[12];
#pragma unroll
    for (int c = 0; c < 24; c += 2) {
      const __half2 v = __floats2half2_rn(hv[hpos(c)], hv[hpos(c + 1)]);
      w[c / 2] = *reinterpret_cast<const uint32_t*>(&v);
    }
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      const uint4 u = make_uint4(w[4 * k], w[4 * k + 1], w[4 * k + 2], w[4 * k + 3]);
      reinterpret_cast<uint4*>(d0)[k] = u;
      reinterpret_cast<uint4*>(d1)[k] = u;
    }
  };

  // ---- embedding h0 = tanh(X.We + be) into both buffers (rows a phase does
  // not update must read the same in either); padded rows and row npad are
  // zero.  Factored: pocket rows start from their cached post-covalent state.
  // We and be are staged in the (not yet used) fragment area for float4
  // broadcast reads.
  float* WE = reinterpret_cast<float*>(WF);   // [F][24] then be[24]
  for (int i = threadIdx.x; i < a.F * 24; i += blockDim.x) WE[i] = a.we[i];
  for (int i = threadIdx.x; i < 24; i += blockDim.x) WE[a.F * 24 + i] = a.be[i];
  __syncthreads();
  if (a.F == 8) {
    // 16-row tiles on the tensor cores: [16 x 8] X . [8 x 24] We in fp16 hi/lo
    // (X = one-hot | role | position/box + 1/2; Xlo.Whi + Xhi.Wlo + Xhi.Whi,
    // ~2^-22 relative, bias as C), k 8..15 zero; lane: rows g, g+8, columns
    // 8nt+2t, 8nt+2t+1 -- the GRU's lane-local layout.
    uint32_t wbh[3], wbl[3];
    float cb[3][2];
#pragma unroll
    for (int nt = 0; nt < 3; ++nt) {
      split2_f16(WE[(2 * t) * 24 + 8 * nt + g], WE[(2 * t + 1) * 24 + 8 * nt + g], wbh[nt], wbl[nt]);
      cb[nt][0] = WE[8 * 24 + 8 * nt + 2 * t];
      cb[nt][1] = WE[8 * 24 + 8 * nt + 2 * t + 1];
    }
    for (int tile = warp; tile < ntiles; tile += kMmaWarps) {
      float v[2][6];
      int rr_row[2];
      uint32_t ah[2], al[2];
#pragma unroll
      for (int rr = 0; rr < 2; ++rr) {
        const int r = tile * 16 + g + 8 * rr;
        rr_row[rr] = r;
        const bool emb = FACT ? r < nL : r < n;
        float2 x = make_float2(0.f, 0.f);
        if (emb) x = __ldg(reinterpret_cast<const float2*>(a.feats + (base + r) * 8 + 2 * t));
        split2_f16(x.x, x.y, ah[rr], al[rr]);
      }
      const uint32_t Ahi[4] = {ah[0], ah[1], 0u, 0u}, Alo[4] = {al[0], al[1], 0u, 0u};
#pragma unroll
      for (int nt = 0; nt < 3; ++nt) {
        float d[4];
        mma_c2<2>(d, Alo, wbh[nt], 0u, cb[nt][0], cb[nt][1]);
        mma_t<2>(d, Ahi, wbl[nt], 0u);
        mma_t<2>(d, Ahi, wbh[nt], 0u);
        v[0][2 * nt] = d[0]; v[0][2 * nt + 1] = d[1];
        v[1][2 * nt] = d[2]; v[1][2 * nt + 1] = d[3];
      }
#pragma unroll
      for (int rr = 0; rr < 2; ++rr) {
        const int r = rr_row[rr];
        const bool emb = FACT ? r < nL : r < n;
        const bool cached = FACT && r >= nLp && r < n;
#pragma unroll
        for (int c = 0; c < 6; ++c) {
          float th;
          if constexpr ((VAR & (8 | 128)) != 0) asm("tanh.approx.f32 %0, %1;" : "=f"(th) : "f"(v[rr][c]));
          else th = fs_tanh(v[rr][c]);
          v[rr][c] = emb ? th : 0.f;
        }
        if (cached) {   // factored: the cached post-covalent state (storage order = this lane's 6 columns)
          const float* src = reinterpret_cast<const float*>(pc + a.off_hcov) +
                             static_cast<int64_t>(a.fact_aff[base + r]) * 24 + 6 * t;
#pragma unroll
          for (int c = 0; c < 6; c += 2) {
            const float2 w = *reinterpret_cast<const float2*>(src + c);
            v[rr][c] = w.x; v[rr][c + 1] = w.y;
          }
        }
#pragma unroll
        for (int c = 0; c < 6; c += 2) {
          *reinterpret_cast<float2*>(Hc + r * 24 + PCOL(c)) = make_float2(v[rr][c], v[rr][c + 1]);
          if constexpr (G16) {
            const int pos = NAT ? 4 * c + 2 * t : PCOL(c);
            const __half2 hv = __floats2half2_rn(v[rr][c], v[rr][c + 1]);
            *reinterpret_cast<__half2*>(Gc + r * 24 + pos) = hv;
            *reinterpret_cast<__half2*>(Gn + r * 24 + pos) = hv;
          } else {
            *reinterpret_cast<float2*>(Hn + r * 24 + PCOL(c)) = make_float2(v[rr][c], v[rr][c + 1]);
          }
        }
      }
    }
    // row npad: the all-zero row of the gathers
    for (int k = threadIdx.x; k < 24; k += blockDim.x) {
      Hc[npad * 24 + k] = 0.f;
      if constexpr (G16) {
        Gc[npad * 24 + k] = __float2half(0.f);
        Gn[npad * 24 + k] = __float2half(0.f);
      } else {
        Hn[npad * 24 + k] = 0.f;
      }
    }
  } else
  for (int i = threadIdx.x; i <= npad; i += blockDim.x) {
    if (FACT && i >= nLp && i < n) {
      const float4* src = reinterpret_cast<const float4*>(
          reinterpret_cast<const float*>(pc + a.off_hcov) + static_cast<int64_t>(a.fact_aff[base + i]) * 24);
      if constexpr (NAT) {
        float hv[24];
#pragma unroll
        for (int k = 0; k < 6; ++k) {
          const float4 v = src[k];
          reinterpret_cast<float4*>(Hc + i * 24)[k] = v;
          hv[4 * k] = v.x; hv[4 * k + 1] = v.y; hv[4 * k + 2] = v.z; hv[4 * k + 3] = v.w;
        }
        store_nat16(Gc + i * 24, Gn + i * 24, hv);
      } else {
#pragma unroll
        for (int k = 0; k < 6; ++k) {
          const float4 v = src[k];
          reinterpret_cast<float4*>(Hc + i * 24)[k] = v;
          if constexpr (G16) {
            const __half2 lo = __floats2half2_rn(v.x, v.y), hi = __floats2half2_rn(v.z, v.w);
            uint2 u;
            u.x = *reinterpret_cast<const uint32_t*>(&lo);
            u.y = *reinterpret_cast<const uint32_t*>(&hi);
            reinterpret_cast<uint2*>(Gc + i * 24)[k] = u;
            reinterpret_cast<uint2*>(Gn + i * 24)[k] = u;
          } else {
            reinterpret_cast<float4*>(Hn + i * 24)[k] = v;
          }
        }
      }
      continue;
    }
    // generic feature width: one row per thread, FFMA
    const bool emb = FACT ? i < nL : i < n;
    float acc[24];
#pragma unroll
    for (int k = 0; k < 24; k += 4) {
      const float4 b4 = *reinterpret_cast<const float4*>(WE + a.F * 24 + k);
      acc[k] = emb ? b4.x : 0.f; acc[k + 1] = emb ? b4.y : 0.f;
      acc[k + 2] = emb ? b4.z : 0.f; acc[k + 3] = emb ? b4.w : 0.f;
    }
    if (emb) {
      const float* x = a.feats + (base + i) * a.F;
      for (int f = 0; f < a.F; ++f) {
        const float xv = x[f];
        const float4* w4 = reinterpret_cast<const float4*>(WE + f * 24);
#pragma unroll
        for (int k = 0; k < 6; ++k) {
          const float4 w = w4[k];
          acc[4 * k] = fmaf(xv, w.x, acc[4 * k]);
          acc[4 * k + 1] = fmaf(xv, w.y, acc[4 * k + 1]);
          acc[4 * k + 2] = fmaf(xv, w.z, acc[4 * k + 2]);
          acc[4 * k + 3] = fmaf(xv, w.w, acc[4 * k + 3]);
        }
      }
    }
    float hv[24];   // storage order
#pragma unroll
    for (int c = 0; c < 24; ++c) {
      float th;
      if constexpr ((VAR & 8) != 0) asm("tanh.approx.f32 %0, %1;" : "=f"(th) : "f"(acc[c]));
      else th = fs_tanh(acc[c]);
      hv[hpos(c)] = emb ? th : 0.f;
    }
    if constexpr (NAT) store_nat16(Gc + i * 24, Gn + i * 24, hv);
#pragma unroll
    for (int k = 0; k < 24; k += 4) {
      const float4 v = make_float4(hv[k], hv[k + 1], hv[k + 2], hv[k + 3]);
      *reinterpret_cast<float4*>(Hc + i * 24 + k) = v;
      if constexpr (NAT) {
        // fp16 copies written above
      } else if constexpr (G16) {
        const __half2 lo = __floats2half2_rn(v.x, v.y), hi = __floats2half2_rn(v.z, v.w);
        uint2 u;
        u.x = *reinterpret_cast<const uint32_t*>(&lo);
        u.y = *reinterpret_cast<const uint32_t*>(&hi);
        *reinterpret_cast<uint2*>(Gc + i * 24 + k) = u;
        *reinterpret_cast<uint2*>(Gn + i * 24 + k) = u;
      } else {
        *reinterpret_cast<float4*>(Hn + i * 24 + k) = v;
      }
    }
  }

  // GRU update of 16 rows held by the warp (lane: rows g and g+8, columns
  // COLS) from their neighbour sums s and states h
  // SPLIT 1/3: bf16 [zr hi | zr lo | hh hi | hh lo]; SPLIT 2: fp16 [zr | hh]
  const uint32_t* zr_hi = WF;
  const uint32_t* zr_lo = WF + kZrWords;
  const uint32_t* hh_hi = WF + (SPLIT == 2 ? kZrWords : 2 * kZrWords);
  const uint32_t* hh_lo = WF + 2 * kZrWords + kHhWords;
  // zs: std::true_type when all 16 rows of the tile have no neighbours (s = 0,
  // e.g. pocket atoms no ligand atom reaches in the non-covalent phase): the
  // s k-tile is skipped in both GEMMs -- exact, the skipped products are zeros
  // slo: std::bool_constant, whether the neighbour sums take a lo pass; with
  // it, slo0 / slo1 say whether row g / g+8 keeps its lo term (a zeroed lo
  // adds exact zeros: a row's result does not depend on its tile-mates)
  auto gru16 = [&](auto zs, auto slo, const float (&sv)[2][6], const float (&h)[2][6], float (&hn)[2][6],
                   bool slo0 = true, bool slo1 = true) {
    constexpr int KT0 = decltype(zs)::value ? 1 : 0;
    // biases as the GEMMs' initial accumulators: columns 8j+2t, 8j+2t+1,
    // one 8-byte load per gate and n-tile
    float cz[6][2];
#pragma unroll
    for (int j = 0; j < 6; ++j) {
      const float2 b2 = *reinterpret_cast<const float2*>(WB + 8 * j + 2 * t);   // z | r
      cz[j][0] = b2.x; cz[j][1] = b2.y;
    }
    uint32_t ahi[3][4], alo[3][4];
    // !SLO: the neighbour sums enter as one fp16 pass (no lo term); they are
    // sums of fp16-rounded rows, so for small sums their own rounding is of
    // the same order (VAR & 32 picks this per row, see kSBig)
    constexpr bool SLO = SPLIT != 2 || decltype(slo)::value;
    // VAR & 64: r*h enters GEMM 2 as one fp16 pass as well (r carries the
    // ~2^-11 error of tanh.approx; the hi/lo split of r*h adds nothing)
    constexpr bool RLO = !(SPLIT == 2 && (VAR & 64));
    constexpr int LOM1 = SLO ? 7 : 6;
    constexpr int LOM2 = (SLO ? 1 : 0) | ((SLO || RLO) ? 2 : 0) | (RLO ? 4 : 0);
    if constexpr (SLO) {
      build_a48<SPLIT>(sv, h, ahi, alo);
      if constexpr (SPLIT == 2 && (VAR & 32) != 0) {
        if (!slo0) { alo[0][0] = 0u; alo[0][2] = 0u; alo[1][0] = 0u; }
        if (!slo1) { alo[0][1] = 0u; alo[0][3] = 0u; alo[1][1] = 0u; }
      }
    } else {
      const float z6[2][6] = {{0.f, 0.f, 0.f, 0.f, 0.f, 0.f}, {0.f, 0.f, 0.f, 0.f, 0.f, 0.f}};
      build_a48<SPLIT>(z6, h, ahi, alo);   // h hi/lo (s slots overwritten below)
      put_a<5>(ahi[0], alo[0], 0, sv[0][0], sv[0][1]);
      put_a<5>(ahi[0], alo[0], 1, sv[1][0], sv[1][1]);
      put_a<5>(ahi[0], alo[0], 2, sv[0][2], sv[0][3]);
      put_a<5>(ahi[0], alo[0], 3, sv[1][2], sv[1][3]);
      put_a<5>(ahi[1], alo[1], 0, sv[0][4], sv[0][5]);
      put_a<5>(ahi[1], alo[1], 1, sv[1][4], sv[1][5]);
      alo[1][0] = 0u; alo[1][1] = 0u;
    }
    float Dzr[6][4];
    gemm48<SPLIT, 6, KT0, LOM1>(Dzr, cz, ahi, alo, zr_hi, zr_lo, lane);
    // D n-tile j holds (row g: cols 8j+2t, 8j+2t+1; row g+8: same)
    // elementwise work on column pairs (2j, 2j+1) with packed fp32 ops
    float z[2][6], rh[2][6];
#pragma unroll
    for (int j = 0; j < 3; ++j)
#pragma unroll
      for (int rr = 0; rr < 2; ++rr) {
        const int c = 2 * j;
        z[rr][c] = Dzr[j][2 * rr]; z[rr][c + 1] = Dzr[j][2 * rr + 1];
        gate_sigmoid2<VAR>(z[rr][c], z[rr][c + 1]);
        rh[rr][c] = Dzr[3 + j][2 * rr]; rh[rr][c + 1] = Dzr[3 + j][2 * rr + 1];
        gate_sigmoid2<VAR>(rh[rr][c], rh[rr][c + 1]);
        fmul2(rh[rr][c], rh[rr][c + 1], h[rr][c], h[rr][c + 1]);
      }
    // A = [s | r*h]: the s part (k-tile 0 and half of k-tile 1) is reused
    constexpr int RS = RLO ? SPLIT : 5;
    put_a<RS>(ahi[1], alo[1], 2, rh[0][0], rh[0][1]);
    put_a<RS>(ahi[1], alo[1], 3, rh[1][0], rh[1][1]);
    put_a<RS>(ahi[2], alo[2], 0, rh[0][2], rh[0][3]);
    put_a<RS>(ahi[2], alo[2], 1, rh[1][2], rh[1][3]);
    put_a<RS>(ahi[2], alo[2], 2, rh[0][4], rh[0][5]);
    put_a<RS>(ahi[2], alo[2], 3, rh[1][4], rh[1][5]);
    if constexpr (!RLO) { alo[1][2] = 0u; alo[1][3] = 0u; }   // (read only when the s part has a lo pass)
    float Dh[3][4], ch[3][2];
#pragma unroll
    for (int j = 0; j < 3; ++j) {
      const float2 b2 = *reinterpret_cast<const float2*>(WB + 48 + 8 * j + 2 * t);
      ch[j][0] = b2.x; ch[j][1] = b2.y;
    }
    gemm48<SPLIT, 3, KT0, LOM2>(Dh, ch, ahi, alo, hh_hi, hh_lo, lane);
#pragma unroll
    for (int rr = 0; rr < 2; ++rr)
#pragma unroll
      for (int j = 0; j < 3; ++j) {
        const int c = 2 * j;
        float u0 = Dh[j][2 * rr], u1 = Dh[j][2 * rr + 1];
        gate_tanh_pre2<VAR>(u0, u1);                       // hh
        fadd2(u0, u1, -h[rr][c], -h[rr][c + 1]);          // hh - h
        ffma2(u0, u1, z[rr][c], z[rr][c + 1], h[rr][c], h[rr][c + 1]);   // h + z (hh - h)
        // padding rows (ok false) evolve too: no CSR row lists them and the
        // pool masks them, so their values are never read
        hn[rr][c] = u0;
        hn[rr][c + 1] = u1;
      }
  };
  auto load_h = [&](int row, float (&h)[6]) {
#pragma unroll
    for (int c = 0; c < 6; c += 2) {
      const float2 hv = *reinterpret_cast<const float2*>(Hc + row * 24 + PCOL(c));
      h[c] = hv.x; h[c + 1] = hv.y;
    }
  };
  auto store_hn = [&](int row, const float (&v)[6]) {
    FS_DCHECK(row >= 0 && row < npad, "gnn state row", row, npad);
    if constexpr (G16) {
      // fp32 state in place (read only by this warp), fp16 copy for the gathers
      // (NAT: natural column order, columns 8j+2t, 8j+2t+1)
#pragma unroll
      for (int c = 0; c < 6; c += 2) {
        *reinterpret_cast<float2*>(Hc + row * 24 + PCOL(c)) = make_float2(v[c], v[c + 1]);
        *reinterpret_cast<__half2*>(Gn + row * 24 + (NAT ? 4 * c + 2 * t : PCOL(c))) = __floats2half2_rn(v[c], v[c + 1]);
      }
    } else {
#pragma unroll
      for (int c = 0; c < 6; c += 2) *reinterpret_cast<float2*>(Hn + row * 24 + PCOL(c)) = make_float2(v[c], v[c + 1]);
    }
  };

  int gstep = 0;
  GPROF(0, 1, clock64());
  for (int ph = 0; ph < 2; ++ph) {
    __syncthreads();
    if (!FACT && ph == 1 && a.dump_hcov) {   // pocket preparation: post-covalent states
      float* o = a.dump_hcov + static_cast<int64_t>(p) * a.dump_ld * 24;
      for (int i = threadIdx.x; i < n * 24; i += blockDim.x) o[i] = Hc[i];
    }
    // factored covalent phase: only the ligand rows move
    const int prow = FACT && ph == 0 ? nLp : npad;
    if (SPLIT == 2) {
      for (int i = threadIdx.x; i < kZrWords + kHhWords; i += blockDim.x) WF[i] = a.wfrag16[ph][i];
    } else {
      for (int i = threadIdx.x; i < kPhaseWords; i += blockDim.x) WF[i] = a.wfrag[ph][i];
    }
    for (int i = threadIdx.x; i < 72; i += blockDim.x) WB[i] = (SPLIT == 2 ? a.wbias16 : a.wbias)[ph][i];
    // NAT: bins and cursors in the (unused) heavy-sum buffer; per sorted slot
    // the row's CSR offset and degree (SOFF, SDEG) in the upper half of the
    // phase-fragment area (SPLIT 2 stages only the lower half)
    int* hst = NAT ? reinterpret_cast<int*>(HS) : hist;
    uint32_t* SOFF = WF + kZrWords + kHhWords;
    uint16_t* SDEG = reinterpret_cast<uint16_t*>(SOFF + npad);
    if (threadIdx.x < NB) hst[threadIdx.x] = 0;
    if (threadIdx.x < 4) CTL[threadIdx.x] = 0;
    const int64_t* rows = ph == 0 ? a.row_cov : a.row_ncov;
    const int32_t* degs = ph == 0 ? a.deg_cov : a.deg_ncov;
    const col_t* colv = ph == 0 ? a.col_cov : a.col_ncov;
    __syncthreads();
    // gather order: counting sort by degree, descending (bin 0: >= kHeavyDeg).
    // Where a row lands never changes its result (its sum has a fixed order,
    // its GRU row is independent of the tile's other rows).
    constexpr int TOPB = NB - 1;   // bin of degree d: TOPB - min(d, TOPB)
    // NAT: a thread's rows (degree, CSR offset) stay in registers from the
    // count to the placement pass (one global round trip per phase)
    constexpr int kKeep = 3;
    const int64_t row0 = n > 0 ? rows[base] : 0;   // the pose's first CSR entry
    int kd[kKeep];
    uint32_t ko[kKeep];
#pragma unroll
    for (int k = 0; k < kKeep; ++k) {
      const int i = threadIdx.x + k * blockDim.x;
      kd[k] = NAT && i < n ? degs[base + i] : 0;
      ko[k] = NAT && i < n ? static_cast<uint32_t>(rows[base + i] - row0) : 0u;
    }
    for (int i = threadIdx.x; i < prow; i += blockDim.x) {
      const int k = (i - static_cast<int>(threadIdx.x)) / static_cast<int>(blockDim.x);
      const int d = NAT && k < kKeep ? (k == 0 ? kd[0] : k == 1 ? kd[1] : kd[2]) : (i < n ? degs[base + i] : 0);
      atomicAdd(&hst[TOPB - min(d, TOPB)], 1);
    }
    __syncthreads();
    if (warp == 0) {   // exclusive scan of the bins into the cursors (5 bins per lane)
      constexpr int PL = (NB + 31) / 32;
      int loc[PL], sum = 0;
#pragma unroll
      for (int k = 0; k < PL; ++k) {
        const int b = lane * PL + k;
        loc[k] = b < NB ? hst[b] : 0;
        sum += loc[k];
      }
      int inc = sum;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int v = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += v;
      }
      int run = inc - sum;
#pragma unroll
      for (int k = 0; k < PL; ++k) {
        const int b = lane * PL + k;
        if (b < NB) hst[NB + b] = run;
        run += loc[k];
      }
    }
    __syncthreads();
    // heavy rows beyond the HS capacity join the first light tiles; which rows
    // those are must be deterministic (heavy and light sums differ in order),
    // so bin 0 is placed in ascending row order by a block prefix count
    const int nh = NAT ? 0 : min(hist[1 + kBins] - hist[kBins], a.heavy_cap);
    if constexpr (!NAT) {
      int run = 0;
      for (int i0 = 0; i0 < prow; i0 += blockDim.x) {
        const int i = i0 + threadIdx.x;
        const bool hv = i < prow && (i < n ? degs[base + i] : 0) >= kHeavyDeg;
        const unsigned m = __ballot_sync(0xffffffffu, hv);
        if (lane == 0) wcnt[warp] = __popc(m);
        __syncthreads();
        int before = 0, total = 0;
        for (int w = 0; w < kMmaWarps; ++w) { const int c = wcnt[w]; before += w < warp ? c : 0; total += c; }
        if (hv) PERM[run + before + __popc(m & ((1u << lane) - 1u))] = static_cast<uint16_t>(i);
        run += total;
        __syncthreads();
      }
    }
    const col_t* cbase = colv + row0;
    for (int i = threadIdx.x; i < prow; i += blockDim.x) {
      const int k = (i - static_cast<int>(threadIdx.x)) / static_cast<int>(blockDim.x);
      const bool kept = NAT && k < kKeep;
      const int d = kept ? (k == 0 ? kd[0] : k == 1 ? kd[1] : kd[2]) : (i < n ? degs[base + i] : 0);
      if (NAT || d < kHeavyDeg) {
        const int pos = atomicAdd(&hst[NB + TOPB - min(d, TOPB)], 1);
        PERM[pos] = static_cast<uint16_t>(i);
        if constexpr (NAT) {
          SOFF[pos] = kept ? (k == 0 ? ko[0] : k == 1 ? ko[1] : ko[2])
                           : (i < n ? static_cast<uint32_t>(rows[base + i] - row0) : 0u);
          SDEG[pos] = static_cast<uint16_t>(d);
        }
      }
    }
    __syncthreads();
    const int nlt = (prow - nh + 15) / 16, nht = (nh + 15) / 16;
    GPROF(11, ph, clock64());   // phase setup + sort done
    const int nitems = nh + nlt + nht;

    for (int step = 0; step < a.k_steps[ph]; ++step) {
      const float* H4 = Hc + 6 * t + ((t & 1) << 1);   // this step's gather bases (acc_row_at)
      const float* H2 = Hc + 6 * t + ((t & 1) ? 0 : 4);
      const __half* G4 = Gc + 6 * t + ((t & 1) << 1);
      const __half* G2 = Gc + 6 * t + ((t & 1) ? 0 : 4);
      // row npad is the all-zero row (CSR padding, exhausted tile rows):
      // adding it is the identity; on the fp32 rows those loads are
      // predicated off (25.4 -> 25.2 ms per 16,384 poses; on the fp16 rows
      // the branch costs more than the wavefronts it saves: 19.8 -> 20.8)
      auto acc = [&](float (&q)[4], float (&d)[2], int j) {
        FS_DCHECK(j >= 0 && j <= npad, "gnn gather row", j, npad);
        if constexpr (!G16) {
          if (j == npad) return;
        }
        if constexpr (G16) acc_row_at16(q, d, G4, G2, j);
        else acc_row_at(q, d, H4, H2, j);
      };
      // Items, handed out in order by a counter: heavy-row sums (-> HS), then
      // the degree-sorted light tiles (gather + GRU), then the heavy tiles
      // (GRU from HS, after every heavy sum is in).
      int* ctr = CTL + (gstep & 1);
      int* hdone = CTL + 2 + (gstep & 1);
#ifdef FS_GNN_PROF
      long long prof_items = 0, prof_gather = 0, prof_claim = 0, prof_gru = 0, prof_lo = 0;
#endif
      GPROF(1 + gstep, 0, clock64());
      if constexpr (NAT) {
        // 16 degree-sorted rows per item; lane l stages slot l & 15 (row k of
        // the tile) for the ldmatrix loads and owns rows g and g+8 in the GRU.
        // Chunk c = the c-th neighbour of every row of the tile; past a row's
        // degree its slot reads the all-zero row npad.  The next item's row
        // metadata and first CSR ids are fetched during this item's GRU, and
        // long rows prefetch their ids two 8-chunk rounds ahead (lanes < 16
        // load chunks q..q+3 of their row, lanes >= 16 chunks q+4..q+7).
        const uint32_t gs = static_cast<uint32_t>(__cvta_generic_to_shared(Gc));
        const uint32_t ga = gs + ((lane >> 4) << 4);   // columns 0-7 / 8-15
        const uint32_t gcl = gs + 32;                  // columns 16-23
        const uint32_t ai = (g == 2 * t ? 0x3C00u : 0u) | (g == 2 * t + 1 ? 0x3C000000u : 0u);   // I16 fragment
        const uint32_t padw = static_cast<uint32_t>(npad) * 0x10001u;
        const int kk = lane & 15, hi4 = (lane >> 4) << 2;
        struct Meta { int rk, dk, ek, nch; const col_t* ck; };
        // (instantiated for padded and packed CSR rows: no per-load branch)
        auto nat_items = [&](auto padded) {
        constexpr bool PADDED = decltype(padded)::value;
        auto meta = [&](int it, Meta& m) {
          const int ks = it * 16 + kk;
          const bool in = it < nitems && ks < prow;
          m.rk = in ? PERM[ks] : npad;
          m.dk = in ? SDEG[ks] : 0;
          m.ck = cbase + (in ? SOFF[ks] : 0u);
          m.ek = PADDED ? ((m.dk + 3) & ~3) : m.dk;
          m.nch = __reduce_max_sync(0xffffffffu, m.dk);
        };
        auto ld4 = [&](const Meta& m, int q) -> uint2 {   // ids q..q+3 of the lane's row
          if constexpr (PADDED) {
            return q < m.ek ? __ldg(reinterpret_cast<const uint2*>(m.ck + q)) : make_uint2(padw, padw);
          } else {
            uint32_t j[4];
#pragma unroll
            for (int u = 0; u < 4; ++u)
              j[u] = q + u < m.ek ? static_cast<uint32_t>(__ldg(m.ck + q + u)) : static_cast<uint32_t>(npad);
            return make_uint2(j[0] | (j[1] << 16), j[2] | (j[3] << 16));
          }
        };
        Meta cur;
        meta(warp, cur);
        // first ids of an item: chunks 0..3 in every lane for rows of <= 4
        // chunks, else lanes >= 16 take chunks 4..7
        auto ld_first = [&](const Meta& m) -> uint2 {
          if (m.nch <= 0) return make_uint2(padw, padw);
          return ld4(m, m.nch > 4 ? hi4 : 0);
        };
        uint2 x = ld_first(cur);
        // long rows: their second 8-chunk round, fetched with the first
        uint2 x2 = cur.nch > 8 ? ld4(cur, 8 + hi4) : make_uint2(padw, padw);
        for (int item = warp; item < nitems;) {
#ifdef FS_GNN_PROF
          ++prof_items;
          const long long prof_t0 = clock64();
#endif
          // claim the next item; its index is read (shuffled) only after the
          // gather, so the atomic's round trip overlaps it
          int next = 0;
          if (lane == 0) next = atomicAdd(ctr, 1) + kMmaWarps;
#ifdef FS_GNN_PROF
          const long long prof_t1 = clock64();
          prof_claim += prof_t1 - prof_t0;
#endif
          float D0[3][4], D1[3][4];
          // chunks (w & 0xffff, w >> 16) into D0, D1; FIRST: the chains' first MMAs (C = 0)
          auto pair = [&](uint32_t w, auto first) {
            const uint32_t i0 = w & 0xffffu, i1 = w >> 16;
            FS_DCHECK(i0 <= static_cast<uint32_t>(npad) && i1 <= static_cast<uint32_t>(npad), "gnn gather row",
                      i0 > i1 ? i0 : i1, npad);
            uint32_t b[4], c[4], e[4];
            ldsm_x4_t(b, ga + i0 * 48u);
            ldsm_x4_t(c, ga + i1 * 48u);
            ldsm_x4_t(e, gcl + (lane < 16 ? i0 : i1) * 48u);
            if constexpr (decltype(first)::value) {
              mma_f16_id0(D0[0], ai, b[0], b[1]);
              mma_f16_id0(D0[1], ai, b[2], b[3]);
              mma_f16_id0(D0[2], ai, e[0], e[1]);
              mma_f16_id0(D1[0], ai, c[0], c[1]);
              mma_f16_id0(D1[1], ai, c[2], c[3]);
              mma_f16_id0(D1[2], ai, e[2], e[3]);
            } else {
              mma_f16_id(D0[0], ai, b[0], b[1]);
              mma_f16_id(D0[1], ai, b[2], b[3]);
              mma_f16_id(D0[2], ai, e[0], e[1]);
              mma_f16_id(D1[0], ai, c[0], c[1]);
              mma_f16_id(D1[1], ai, c[2], c[3]);
              mma_f16_id(D1[2], ai, e[2], e[3]);
            }
          };
          const int nch = cur.nch;
          if (nch == 0) {
#pragma unroll
            for (int j = 0; j < 3; ++j)
#pragma unroll
              for (int e = 0; e < 4; ++e) { D0[j][e] = 0.f; D1[j][e] = 0.f; }
          } else if (nch <= 4) {   // one round, ids 0..3 in every lane
            pair(x.x, std::true_type{});
            if (nch > 2) pair(x.y, std::false_type{});
          } else {
            const uint2 y0 = x2;
            uint2 o;
            o.x = __shfl_xor_sync(0xffffffffu, x.x, 16);
            o.y = __shfl_xor_sync(0xffffffffu, x.y, 16);
            {
              const uint2 wl = lane < 16 ? x : o, wh = lane < 16 ? o : x;   // chunks 0..3, 4..7
              pair(wl.x, std::true_type{});
              pair(wl.y, std::false_type{});   // (nch > 4)
              pair(wh.x, std::false_type{});
              if (nch > 6) pair(wh.y, std::false_type{});
            }
            if (nch > 8) {   // long rows: ids two rounds ahead
              x = y0;
              uint2 y = nch > 16 ? ld4(cur, 16 + hi4) : make_uint2(padw, padw);
              int q = 8;
              for (; q + 8 <= nch; q += 8) {   // full rounds: four unconditional pairs
                const uint2 z = q + 16 < nch ? ld4(cur, q + 16 + hi4) : make_uint2(padw, padw);
                o.x = __shfl_xor_sync(0xffffffffu, x.x, 16);
                o.y = __shfl_xor_sync(0xffffffffu, x.y, 16);
                const uint2 wl = lane < 16 ? x : o, wh = lane < 16 ? o : x;   // chunks q..q+3, q+4..q+7
                pair(wl.x, std::false_type{});
                pair(wl.y, std::false_type{});
                pair(wh.x, std::false_type{});
                pair(wh.y, std::false_type{});
                x = y;
                y = z;
              }
              if (q < nch) {   // the last, partial round
                o.x = __shfl_xor_sync(0xffffffffu, x.x, 16);
                o.y = __shfl_xor_sync(0xffffffffu, x.y, 16);
                const uint2 wl = lane < 16 ? x : o, wh = lane < 16 ? o : x;
                pair(wl.x, std::false_type{});
                if (q + 2 < nch) pair(wl.y, std::false_type{});
                if (q + 4 < nch) pair(wh.x, std::false_type{});
                if (q + 6 < nch) pair(wh.y, std::false_type{});
              }
            }
          }
          float sv[2][6];
#pragma unroll
          for (int j = 0; j < 3; ++j) {
            fadd2(D0[j][0], D0[j][1], D1[j][0], D1[j][1]);
            fadd2(D0[j][2], D0[j][3], D1[j][2], D1[j][3]);
            sv[0][2 * j] = D0[j][0]; sv[0][2 * j + 1] = D0[j][1];
            sv[1][2 * j] = D0[j][2]; sv[1][2 * j + 1] = D0[j][3];
          }
#ifdef FS_GNN_PROF
          const long long prof_t2 = clock64() + (sv[0][0] == 1e30f ? 1 : 0);
          prof_gather += prof_t2 - prof_t1;
#endif
          const int r0 = __shfl_sync(0xffffffffu, cur.rk, g), r1 = __shfl_sync(0xffffffffu, cur.rk, g + 8);
          next = __shfl_sync(0xffffffffu, next, 0);
          Meta nm;   // the next item's rows and first ids, in flight during the GRU
          meta(next, nm);
          const uint2 nx = ld_first(nm);
          const uint2 nx2 = nm.nch > 8 ? ld4(nm, 8 + hi4) : make_uint2(padw, padw);
          float h[2][6], hn[2][6];
          load_h(r0, h[0]);
          load_h(r1, h[1]);
          if (nch == 0) {
            gru16(std::true_type{}, std::false_type{}, sv, h, hn);
          } else if constexpr ((VAR & 32) != 0) {
            // a row's sums take one fp16 pass while all its |s| <= kSBig (the
            // row's lo term is zeroed); the tile runs the lo MMAs only if
            // some row keeps its lo term
            float m0 = 0.f, m1 = 0.f;
#pragma unroll
            for (int c = 0; c < 6; ++c) { m0 = fmaxf(m0, fabsf(sv[0][c])); m1 = fmaxf(m1, fabsf(sv[1][c])); }
            // a row's 24 sums sit in its 4 lanes (bits 4g..4g+3 of a ballot)
            const unsigned q0 = __ballot_sync(0xffffffffu, m0 > kSBig), q1 = __ballot_sync(0xffffffffu, m1 > kSBig);
            const bool b0 = (q0 >> (4 * g)) & 15u, b1 = (q1 >> (4 * g)) & 15u;
            if (q0 | q1) {
#ifdef FS_GNN_PROF
              ++prof_lo;
#endif
              gru16(std::false_type{}, std::true_type{}, sv, h, hn, b0, b1);
            } else {
              gru16(std::false_type{}, std::false_type{}, sv, h, hn);
            }
          } else {
            gru16(std::false_type{}, std::true_type{}, sv, h, hn);
          }
          if (r0 < npad) store_hn(r0, hn[0]);
          if (r1 < npad) store_hn(r1, hn[1]);
#ifdef FS_GNN_PROF
          prof_gru += clock64() - prof_t2 + (hn[0][0] == 1e30f ? 1 : 0);
#endif
          cur = nm;
          x = nx;
          x2 = nx2;
          item = next;
        }
        };
        if (a.ids_padded) nat_items(std::true_type{});
        else nat_items(std::false_type{});
      } else
      for (int item = warp; item < nitems;) {
#ifdef FS_GNN_PROF
        ++prof_items;
#endif
        // claim the next item now: the counter's round trip overlaps this
        // item's work (items are claimed in increasing order, so a warp
        // spinning in a heavy tile never holds an unprocessed heavy sum)
        int next = 0;
        if (lane == 0) next = atomicAdd(ctr, 1) + kMmaWarps;
        if (item < nh) {
          // one heavy row: lane (q = lane/4, t) sums neighbours q, q+8, ...
          const int row = PERM[item];
          const int d = degs[base + row];
          const col_t* c = colv + rows[base + row];
          float sq[4] = {0.f, 0.f, 0.f, 0.f}, sd[2] = {0.f, 0.f};
          if (a.ids_padded) {
            // rows padded to 4 ids (zero row npad): lane group g takes ids
            // 4g..4g+3 of every 32, one 8-byte load
            const int e = (d + 3) & ~3;
            for (int q = 4 * g; q < e; q += 32) {
              const uint2 v = __ldg(reinterpret_cast<const uint2*>(c + q));
              const int j[4] = {static_cast<int>(v.x & 0xffffu), static_cast<int>(v.x >> 16),
                                static_cast<int>(v.y & 0xffffu), static_cast<int>(v.y >> 16)};
#pragma unroll
              for (int u = 0; u < 4; ++u) acc(sq, sd, j[u]);
            }
          } else {
            for (int q = g; q < d; q += 32) {
              int j[4];
#pragma unroll
              for (int u = 0; u < 4; ++u) j[u] = q + 8 * u < d ? __ldg(c + q + 8 * u) : npad;
#pragma unroll
              for (int u = 0; u < 4; ++u) acc(sq, sd, j[u]);
            }
          }
          float s6[6] = {sq[0], sq[1], sq[2], sq[3], sd[0], sd[1]};   // storage order
#pragma unroll
          for (int k = 0; k < 6; ++k) {
            float v = s6[k];
            v += __shfl_xor_sync(0xffffffffu, v, 4);
            v += __shfl_xor_sync(0xffffffffu, v, 8);
            v += __shfl_xor_sync(0xffffffffu, v, 16);
            s6[k] = v;
          }
          if (g == 0) {
            FS_DCHECK(item < a.heavy_cap, "gnn heavy slot", item, a.heavy_cap);
            float* b = HS + item * 24 + 6 * t;
            *reinterpret_cast<float4*>(b + ((t & 1) << 1)) = make_float4(s6[0], s6[1], s6[2], s6[3]);
            *reinterpret_cast<float2*>(b + ((t & 1) ? 0 : 4)) = make_float2(s6[4], s6[5]);
          }
          __syncwarp();
          if (lane == 0) { __threadfence_block(); atomicAdd(hdone, 1); }
        } else if (item < nh + nlt) {
          // 16 degree-sorted light rows; lane (g, t) owns rows g and g+8.
          // Exhausted slots read the all-zero row `npad` (x + 0 == x, so the
          // sums stay exactly CSR-ordered).  The sums land in the lane's
          // A-fragment positions and feed the GRU directly.
          const int k0 = nh + (item - nh) * 16 + g, k1 = k0 + 8;
          const int r0 = k0 < prow ? PERM[k0] : npad, r1 = k1 < prow ? PERM[k1] : npad;
          const int d0 = r0 < n ? degs[base + r0] : 0, d1 = r1 < n ? degs[base + r1] : 0;
          const col_t* c0 = colv + (r0 < n ? rows[base + r0] : 0);
          const col_t* c1 = colv + (r1 < n ? rows[base + r1] : 0);
          float sq[2][4] = {{0.f, 0.f, 0.f, 0.f}, {0.f, 0.f, 0.f, 0.f}}, sd[2][2] = {{0.f, 0.f}, {0.f, 0.f}};
          if (a.ids_padded) {
            // rows padded to 4 ids with the zero row `npad` (graph_csr.cu):
            // ids come 4 at a time; past a row's padded extent the lane reads
            // row npad (x + 0 == x: sums stay exactly CSR-ordered)
            const int e0 = (d0 + 3) & ~3, e1 = (d1 + 3) & ~3;
            const int nch = max(e0, e1) >> 2;          // 4-id chunks
            // ids are software-pipelined one 8-id round ahead: the global
            // (L2) latency of round k+1 overlaps the gathers of round k
            const uint32_t padw = static_cast<uint32_t>(npad) * 0x10001u;
            auto ld = [&](const col_t* c, int q, int e) {
              return q < e ? __ldg(reinterpret_cast<const uint2*>(c + q)) : make_uint2(padw, padw);
            };
            auto gather4 = [&](int r, uint2 v) {
              acc(sq[r], sd[r], static_cast<int>(v.x & 0xffffu));
              acc(sq[r], sd[r], static_cast<int>(v.x >> 16));
              acc(sq[r], sd[r], static_cast<int>(v.y & 0xffffu));
              acc(sq[r], sd[r], static_cast<int>(v.y >> 16));
            };
            uint2 x0 = ld(c0, 0, e0), x1 = ld(c1, 0, e1), y0 = ld(c0, 4, e0), y1 = ld(c1, 4, e1);
            for (int k = 0; k < nch; k += 2) {
              const int qn = 4 * (k + 2);
              const uint2 nx0 = ld(c0, qn, e0), nx1 = ld(c1, qn, e1);
              const uint2 ny0 = ld(c0, qn + 4, e0), ny1 = ld(c1, qn + 4, e1);
              gather4(0, x0);
              gather4(1, x1);
              if (k + 1 < nch) {
                gather4(0, y0);
                gather4(1, y1);
              }
              x0 = nx0; x1 = nx1; y0 = ny0; y1 = ny1;
            }
          } else {
            // packed CSR (rows built from reference edge lists): one id per load
            const int dm = max(d0, d1);
            for (int q = 0; q < dm; q += 4) {
              int j0[4], j1[4];
#pragma unroll
              for (int u = 0; u < 4; ++u) j0[u] = q + u < d0 ? __ldg(c0 + q + u) : npad;
#pragma unroll
              for (int u = 0; u < 4; ++u) j1[u] = q + u < d1 ? __ldg(c1 + q + u) : npad;
#pragma unroll
              for (int u = 0; u < 4; ++u) {
                acc(sq[0], sd[0], j0[u]);
                acc(sq[1], sd[1], j1[u]);
              }
            }
          }
          float sv[2][6];
          frag_order(sq[0], sd[0], t, sv[0]);
          frag_order(sq[1], sd[1], t, sv[1]);
          float h[2][6], hn[2][6];
          load_h(r0, h[0]);
          load_h(r1, h[1]);
          // (SPLIT 2 only: on the 3-pass path the second GRU instantiation
          // costs more than the skipped MMAs save, 25.15 -> 25.21 ms)
          if constexpr (SPLIT == 2) {
            if (__all_sync(0xffffffffu, d0 == 0 && d1 == 0)) gru16(std::true_type{}, std::true_type{}, sv, h, hn);
            else gru16(std::false_type{}, std::true_type{}, sv, h, hn);
          } else {
            gru16(std::false_type{}, std::true_type{}, sv, h, hn);
          }
          if (r0 < npad) store_hn(r0, hn[0]);
          if (r1 < npad) store_hn(r1, hn[1]);
        } else {
          // heavy tile: 16 heavy rows' sums from HS
          const int i0 = (item - nh - nlt) * 16 + g, i1 = i0 + 8;
          const int r0 = i0 < nh ? PERM[i0] : npad, r1 = i1 < nh ? PERM[i1] : npad;
          if (lane == 0) {
            while (*reinterpret_cast<volatile int*>(hdone) < nh) { }
            __threadfence_block();
          }
          __syncwarp();
          float sv[2][6], h[2][6], hn[2][6];
#pragma unroll
          for (int c = 0; c < 6; c += 2) {
            const float2 v0 = i0 < nh ? *reinterpret_cast<const float2*>(HS + i0 * 24 + PCOL(c)) : make_float2(0.f, 0.f);
            const float2 v1 = i1 < nh ? *reinterpret_cast<const float2*>(HS + i1 * 24 + PCOL(c)) : make_float2(0.f, 0.f);
            sv[0][c] = v0.x; sv[0][c + 1] = v0.y;
            sv[1][c] = v1.x; sv[1][c + 1] = v1.y;
          }
          load_h(r0, h[0]);
          load_h(r1, h[1]);
          gru16(std::false_type{}, std::true_type{}, sv, h, hn);
          if (r0 < npad) store_hn(r0, hn[0]);
          if (r1 < npad) store_hn(r1, hn[1]);
        }
        item = __shfl_sync(0xffffffffu, next, 0);
      }
#ifdef FS_GNN_PROF
      GPROF(1 + gstep, 1, clock64());
      GPROF(1 + gstep, 2, prof_items);
      GPROF(1 + gstep, 3, prof_gather);
      GPROF(1 + gstep, 4, prof_claim);
      GPROF(1 + gstep, 5, prof_gru);
      GPROF(1 + gstep, 6, prof_lo);
#endif
      // counters of the next step (last used two steps ago)
      if (threadIdx.x == 0) { CTL[(gstep + 1) & 1] = 0; CTL[2 + ((gstep + 1) & 1)] = 0; }
      ++gstep;
      __syncthreads();
      if constexpr (G16) {
        __half* tg = Gc; Gc = Gn; Gn = tg;
      } else {
        float* tmp = Hc; Hc = Hn; Hn = tmp;
      }
    }
  }
  GPROF(11, 2, clock64());   // pool start
  float* RED = Hn;   // [warps][128] (+ [warps][128] doubles), written only after every warp is done with the staged fragments

  // ---- gated gather + mean pool: [gate|val] = h.[Gg|Gf] (K 24->32, N 256) ----
  float acc[16][2];
#pragma unroll
  for (int j = 0; j < 16; ++j) { acc[j][0] = 0.f; acc[j][1] = 0.f; }
  // gather fragments: stage into the (now free) neighbour-sum buffer when it
  // is large enough, else read them through L1
  // SPLIT 2: one fp16 fragment set (the layout of the bf16 "hi" half)
  const uint32_t* gsrc = SPLIT == 2 ? a.gfrag16 : a.gfrag;
  const float* gb = SPLIT == 2 ? a.gbias16 : a.gbias;
  if (hrows * 24 >= kGatherWords + 256) {
    uint32_t* gs = reinterpret_cast<uint32_t*>(Hn);
    const int gw = SPLIT == 2 ? kGatherWords / 2 : kGatherWords;
    for (int i = threadIdx.x; i < gw; i += blockDim.x) gs[i] = gsrc[i];
    float* gbs = reinterpret_cast<float*>(gs + kGatherWords);
    for (int i = threadIdx.x; i < 256; i += blockDim.x) gbs[i] = gb[i];
    gsrc = gs;
    gb = gbs;
  }
  __syncthreads();
  const uint32_t* g_hi = gsrc;
  const uint32_t* g_lo = gsrc + kGatherWords / 2;
  // items = (tile, column quarter): 4 x ntiles items spread the pool over the
  // warps in finer rounds (ntiles is ~4 x the warp count: whole-tile items
  // left a round with one busy warp)
  for (int pit = warp; pit < kPoolSplit * ntiles; pit += kMmaWarps) {
    const int tile = pit / kPoolSplit, half = pit % kPoolSplit;
    float h[2][6];
#pragma unroll
    for (int rr = 0; rr < 2; ++rr) {
      const int row = tile * 16 + g + 8 * rr;
#pragma unroll
      for (int c = 0; c < 6; c += 2) {
        const float2 hv = *reinterpret_cast<const float2*>(Hc + row * 24 + PCOL(c));
        h[rr][c] = hv.x; h[rr][c + 1] = hv.y;
      }
    }
    // k-tile 0: h[0..15]; k-tile 1: h[16..23] | zero padding.  With the fp16
    // weights (SPLIT 2) the pool takes h as one fp16 pass (PS 5): its
    // rounding is per node and the mean over the pose's nodes averages it,
    // unlike the recurrent GRU inputs
    constexpr int PS = SPLIT == 2 ? 5 : SPLIT;
    uint32_t ahi[2][4], alo[2][4];
    put_a<PS>(ahi[0], alo[0], 0, h[0][0], h[0][1]);
    put_a<PS>(ahi[0], alo[0], 1, h[1][0], h[1][1]);
    put_a<PS>(ahi[0], alo[0], 2, h[0][2], h[0][3]);
    put_a<PS>(ahi[0], alo[0], 3, h[1][2], h[1][3]);
    put_a<PS>(ahi[1], alo[1], 0, h[0][4], h[0][5]);
    put_a<PS>(ahi[1], alo[1], 1, h[1][4], h[1][5]);
    const bool v0 = valid(tile * 16 + g), v1 = valid(tile * 16 + g + 8);
    // FULL: every row of the tile holds a node and no per-node dump: no masks
    // and no dump stores in the unrolled column loop (all tiles but the last,
    // on the scoring path)
    auto columns = [&](auto full) {
    constexpr bool FULL = decltype(full)::value;
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      if (j / (16 / kPoolSplit) != half) continue;   // this item's column groups
      // biases enter as the first MMA's C operand
      float Dg[4], Dv[4];
      {
        const float2 bg = *reinterpret_cast<const float2*>(gb + 8 * j + 2 * t);
        const float2 bv = *reinterpret_cast<const float2*>(gb + 128 + 8 * j + 2 * t);
        const float Cg[4] = {bg.x, bg.y, bg.x, bg.y}, Cv[4] = {bv.x, bv.y, bv.x, bv.y};
        // k 0..15: m16n8k16; k 16..23: m16n8k8 (the k16 fragments' first
        // registers; rows 24..31 are zero padding)
        const uint2 bgh = *reinterpret_cast<const uint2*>(g_hi + (j * 32 + lane) * 2);
        const uint2 bvh = *reinterpret_cast<const uint2*>(g_hi + ((16 + j) * 32 + lane) * 2);
        if (SPLIT == 3) {
          const uint2 bgl = *reinterpret_cast<const uint2*>(g_lo + (j * 32 + lane) * 2);
          const uint2 bvl = *reinterpret_cast<const uint2*>(g_lo + ((16 + j) * 32 + lane) * 2);
          mma_bf16_c(Dg, alo[0], bgh.x, bgh.y, Cg);
          mma_bf16_c(Dv, alo[0], bvh.x, bvh.y, Cv);
          mma_bf16(Dg, ahi[0], bgl.x, bgl.y);
          mma_bf16(Dv, ahi[0], bvl.x, bvl.y);
          mma_bf16(Dg, ahi[0], bgh.x, bgh.y);
          mma_bf16(Dv, ahi[0], bvh.x, bvh.y);
        } else if (SPLIT == 2) {
          mma_f16_c(Dg, ahi[0], bgh.x, bgh.y, Cg);
          mma_f16_c(Dv, ahi[0], bvh.x, bvh.y, Cv);
        } else {
          mma_bf16_c(Dg, ahi[0], bgh.x, bgh.y, Cg);
          mma_bf16_c(Dv, ahi[0], bvh.x, bvh.y, Cv);
        }
      }
      {
        const uint32_t bgh = g_hi[((32 + j) * 32 + lane) * 2];
        const uint32_t bvh = g_hi[((32 + 16 + j) * 32 + lane) * 2];
        if (SPLIT == 3) {
          const uint32_t bgl = g_lo[((32 + j) * 32 + lane) * 2];
          const uint32_t bvl = g_lo[((32 + 16 + j) * 32 + lane) * 2];
          mma_bf16_k8(Dg, alo[1][0], alo[1][1], bgh);
          mma_bf16_k8(Dv, alo[1][0], alo[1][1], bvh);
          mma_bf16_k8(Dg, ahi[1][0], ahi[1][1], bgl);
          mma_bf16_k8(Dv, ahi[1][0], ahi[1][1], bvl);
        }
        mma_t_k8<SPLIT>(Dg, ahi[1][0], ahi[1][1], bgh);
        mma_t_k8<SPLIT>(Dv, ahi[1][0], ahi[1][1], bvh);
      }
      {
        // rows g (D[0], D[1]) and g+8 (D[2], D[3]), columns 8j+2t, +1
        if constexpr (SPLIT == 2 && (VAR & 8) != 0) {
          // VAR & 8: one tanh.approx.f16x2 per pair of activations and the
          // gate x value product in fp16 (half the MUFU work of the pool,
          // which is MUFU-bound; each node's term is rounded once and the
          // mean over the pose's nodes averages it)
          auto th2 = [](float u0, float u1) {
            const __half2 x = __floats2half2_rn(u0, u1);
            uint32_t xi = *reinterpret_cast<const uint32_t*>(&x), yi;
            asm("tanh.approx.f16x2 %0, %1;" : "=r"(yi) : "r"(xi));
            return *reinterpret_cast<const __half2*>(&yi);
          };
          const __half2 hh5 = __float2half2_rn(0.5f);
          const __half2 p01 = __hmul2(__hfma2(th2(Dg[0], Dg[1]), hh5, hh5), th2(Dv[0], Dv[1]));
          const __half2 p23 = __hmul2(__hfma2(th2(Dg[2], Dg[3]), hh5, hh5), th2(Dv[2], Dv[3]));
          const float2 f01 = __half22float2(p01), f23 = __half22float2(p23);
          Dg[0] = f01.x; Dg[1] = f01.y; Dg[2] = f23.x; Dg[3] = f23.y;
        } else if constexpr (SPLIT == 2) {
          // one MUFU.TANH per activation (2^-10.7): sigmoid(x) = (1 + tanh(x/2)) / 2
          // (the fp16 pool weights carry the 1/2)
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            float tg, tv;
            asm("tanh.approx.f32 %0, %1;" : "=f"(tg) : "f"(Dg[e]));
            asm("tanh.approx.f32 %0, %1;" : "=f"(tv) : "f"(Dv[e]));
            Dg[e] = fmaf(0.5f, tg, 0.5f);
            Dv[e] = tv;
          }
        } else {
          sigmoid_pre2(Dg[0], Dg[1]); sigmoid_pre2(Dg[2], Dg[3]);
          tanh_pre2(Dv[0], Dv[1]); tanh_pre2(Dv[2], Dv[3]);
        }
        if constexpr (!(SPLIT == 2 && (VAR & 8) != 0)) {
          fmul2(Dg[0], Dg[1], Dv[0], Dv[1]);
          fmul2(Dg[2], Dg[3], Dv[2], Dv[3]);
        }
        const float x00 = FULL || v0 ? Dg[0] : 0.f, x01 = FULL || v0 ? Dg[1] : 0.f;
        const float x10 = FULL || v1 ? Dg[2] : 0.f, x11 = FULL || v1 ? Dg[3] : 0.f;
        float s0 = x00, s1 = x01;
        fadd2(s0, s1, x10, x11);
        fadd2(acc[j][0], acc[j][1], s0, s1);
        if (!FULL && !FACT && a.dump_f) {   // pocket preparation: per-node pool terms
          float* o = a.dump_f + (static_cast<int64_t>(p) * a.dump_ld + tile * 16 + g) * 128 + 8 * j + 2 * t;
          if (v0) { o[0] = x00; o[1] = x01; }
          if (v1) { o[8 * 128] = x10; o[8 * 128 + 1] = x11; }
        }
      }
    }
    };
    if (__all_sync(0xffffffffu, v0 && v1) && (FACT || !a.dump_f)) columns(std::true_type{});
    else columns(std::false_type{});
  }
  // reduce over g (lane bits 2..4), fixed tree
#pragma unroll
  for (int j = 0; j < 16; ++j)
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      float v = acc[j][e];
      v += __shfl_xor_sync(0xffffffffu, v, 4);
      v += __shfl_xor_sync(0xffffffffu, v, 8);
      v += __shfl_xor_sync(0xffffffffu, v, 16);
      acc[j][e] = v;
    }
  __syncthreads();
  if (g == 0) {
#pragma unroll
    for (int j = 0; j < 16; ++j)
#pragma unroll
      for (int e = 0; e < 2; ++e) RED[warp * 128 + 8 * j + 2 * t + e] = acc[j][e];
  }
  double* RED2 = reinterpret_cast<double*>(RED + kMmaWarps * 128);   // [warps][128] (factored only)
  if constexpr (FACT) {
    // cached pool terms of the touched pocket nodes (to be replaced by their
    // recomputed ones): warp w sums rows nLp+w, nLp+w+16, ...; lane owns 4 columns
    const float* f = reinterpret_cast<const float*>(pc + a.off_f);
    double cs[4] = {0.0, 0.0, 0.0, 0.0};
    for (int r = nLp + warp; r < n; r += kMmaWarps) {
      const float4 v = __ldg(reinterpret_cast<const float4*>(f + static_cast<int64_t>(a.fact_aff[base + r]) * 128) + lane);
      cs[0] += v.x; cs[1] += v.y; cs[2] += v.z; cs[3] += v.w;
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) RED2[warp * 128 + 4 * lane + k] = cs[k];
  }
  __syncthreads();
  if (threadIdx.x < 128) {
    float tot = 0.f;
    for (int w = 0; w < kMmaWarps; ++w) tot += RED[w * 128 + threadIdx.x];
    GPROF(10, 0, clock64());
    if constexpr (FACT) {
      // untouched pocket nodes: cached total minus the touched ones' cached terms
      double corr = reinterpret_cast<const double*>(pc + a.off_T)[threadIdx.x];
      for (int w = 0; w < kMmaWarps; ++w) corr -= RED2[w * 128 + threadIdx.x];
      const int n_all = *reinterpret_cast<const int32_t*>(pc + a.off_n) + nL;
      lat[threadIdx.x] = static_cast<float>((corr + static_cast<double>(tot)) / static_cast<double>(max(n_all, 1)));
    } else {
      lat[threadIdx.x] = tot / static_cast<float>(max(n, 1));
    }
  }
}

#ifdef FS_GNN_PROF
extern "C" int fs_debug_gnn_prof(void* host) {
  return cudaMemcpyFromSymbol(host, fs_gnn_prof_buf, sizeof(fs_gnn_prof_buf)) == cudaSuccess ? 0 : -3;
}
#endif

static size_t gnn_smem_bytes(int max_nodes, int heavy_cap) {
  const int npad = (max_nodes + 15) / 16 * 16;
  const int hrows = npad + 1 > kMaxMmaWarps * 16 ? npad + 1 : kMaxMmaWarps * 16;
  return static_cast<size_t>(2 * hrows + heavy_cap) * 24 * 4 + kPhaseWords * 4 + 72 * 4 + kCtlWords * 4 +
         static_cast<size_t>(npad) * 2 + 64;
}
constexpr size_t kSmemLimit = 227 * 1024;
constexpr int kMaxHeavy = 64;

// The heavy-row capacity is a constant: which rows take the heavy path (and so
// their summation order) must not depend on the batch a pose is scored in.
size_t gnn_mma_smem_bytes(int max_nodes) { return gnn_smem_bytes(max_nodes, kMaxHeavy); }

bool gnn_mma_fits(int max_nodes) { return gnn_mma_smem_bytes(max_nodes) <= kSmemLimit; }

int gnn_mma_max_nodes() {
  int n = 16;
  while (gnn_mma_fits(n + 16)) n += 16;
  return n;
}

template <int SPLIT, bool FACT, int WARPS, int VAR = 0>
static int launch_gnn_mma_t(const GnnMmaArgs& a, int n_poses, size_t smem, cudaStream_t st) {
  FS_CUDA_CHECK(cudaFuncSetAttribute(gnn_mma_kernel<SPLIT, FACT, WARPS, VAR>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  gnn_mma_kernel<SPLIT, FACT, WARPS, VAR><<<n_poses, WARPS * 32, smem, st>>>(a);
  FS_LAUNCH_CHECK();
  return FS_OK;
}

// FS_PREC_BF16 (SPLIT 2) variant bits: 1 tanh.approx.f32 gates, 2 f16x2 gates,
// 4 fp16 gather copies, 8 f16x2 pool + approximate embedding tanh, 16
// tensor-core neighbour sums, 32 one-pass fp16 sums for |s| <= kSBig, 64 one-pass
// r*h, 128 approximate (tanh.approx.f32) embedding tanh.  Shipped: 245 =
// 1|4|16|32|64|128 (profiles/r02/gnn_variants.md).
// Round-2 midpoint ran VAR 6: neighbour gathers from fp16 copies of
// the node states (half the shared-memory bytes of the fp32 rows: 21.7 ->
// 20.1 ms per 16,384 poses) and one tanh.approx.f16x2 per pair of gate
// activations (-> 19.8 ms); config-1 score error vs the oracle 1.03e-3 max
// relative (1.33e-3 before; profiles/r02/gnn_variants.md)
#ifdef FS_GNN_WARPS
constexpr int kSplit2Warps = FS_GNN_WARPS;
#else
constexpr int kSplit2Warps = 16;
#endif
#ifdef FS_GNN_WARPS3
constexpr int kSplit3Warps = FS_GNN_WARPS3;
#else
constexpr int kSplit3Warps = 20;
#endif
#ifdef FS_GNN_VAR
constexpr int kSplit2Var = FS_GNN_VAR;   // A/B builds (build_native FS_BUILD_TAG / FS_EXTRA_FLAGS)
#else
constexpr int kSplit2Var = 245;
#endif

int launch_gnn_mma(const GnnMmaArgs& a_in, int split, int n_poses, int max_nodes, cudaStream_t st) {
  if (n_poses <= 0) return FS_OK;
  if (!gnn_mma_fits(max_nodes)) return FS_ECAPACITY;
  GnnMmaArgs a = a_in;
  a.heavy_cap = kMaxHeavy;
  const size_t smem = gnn_mma_smem_bytes(max_nodes);
  if (split == 2) {
    if (!a.wfrag16[0] || !a.wfrag16[1] || !a.gfrag16) return FS_EINVAL;
    // NAT row metadata (6 bytes per row) in the upper half of the fragment area
    if ((kSplit2Var & 16) && (max_nodes + 15) / 16 * 16 * 6 > (kPhaseWords - kZrWords - kHhWords) * 4)
      return FS_ECAPACITY;
    if (a.fact_cnt) return launch_gnn_mma_t<2, true, kSplit2Warps, kSplit2Var>(a, n_poses, smem, st);
    return launch_gnn_mma_t<2, false, kSplit2Warps, kSplit2Var>(a, n_poses, smem, st);
  }
  if (split != 3) return FS_EINVAL;
  if (a.fact_cnt) return launch_gnn_mma_t<3, true, kSplit3Warps>(a, n_poses, smem, st);
  return launch_gnn_mma_t<3, false, kSplit3Warps>(a, n_poses, smem, st);
}

}  // namespace fs
