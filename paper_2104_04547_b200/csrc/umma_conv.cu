// tcgen05 (UMMA) implicit-GEMM Conv3d chain of the default voxel head:
//   conv1 8->32 k5, conv2 32->32 k3 (+relu+2^3 max-pool), conv3 32->64 k3,
//   conv4 64->64 k3 (+relu +residual h3 +2^3 max-pool)   (models.py:300-313)
// bf16 operands, fp32 accumulation in TMEM, bias/ReLU/residual/pool fused in
// the epilogue.  Reference op: conv3d (autodiff.py:208-232), cross-
// correlation, stride 1, zero "same" padding.
//
// im2col-free design.  Every output plane d is one or two M=128 tiles whose
// rows are output voxels (8 consecutive w) x 16 row groups ((h, pose)).  The
// padded input planes are staged by TMA into a shared-memory ring laid out
// chunk-major: [8-channel chunk][h+2r][pose][w+2r] x 16 bytes (zero padding
// comes from TMA out-of-bounds fill).  In that layout the A operand of
// kernel offset (kh,kw) is just a *shifted* K-major no-swizzle UMMA
// descriptor: core-matrix rows (8 w) are 16 B apart, row groups (h,pose) are
// SBO = (w+2r)*16 B apart, the two K chunks of one MMA are LBO apart.
//
// Plane-stacked N.  Input plane q feeds the KS output planes d = q-KS+1..q
// (kernel plane kd = q-d).  Their weights are stored side by side along N
// ([kd descending][cout]), so ONE MMA per (kh,kw,chunk) step contracts the
// staged A tile against all of them: N = cout x (#output planes), up to 160
// (conv1) / 96 (conv2) / 192 (conv3).  Each A tile is read from shared
// memory once per input plane instead of once per (input, output) plane
// pair -- the 32-channel layers were bound by exactly those A re-reads
// (4 KB of operand per 131 kFLOP MMA).  Output planes accumulate in a ring
// of kSlots TMEM slots (d mod kSlots, contiguous columns, so a stacked MMA
// writes consecutive slots); the epilogue drains a finished plane, zeroes
// its slot with tcgen05.st (so every MMA accumulates) and hands it back.
//   16^3 layers: one pose per tile, 2 tiles (w halves) per plane.
//   8^3 layers : two poses per tile, h rows of the pair interleaved (the TMA
//                box spans (w, pose, h) so its dense fill is the interleave).
// Warp roles (192 threads): warp0 = TMA producer, warp1 = TMEM owner + single
// thread UMMA issuer, warps2-5 = epilogue (TMEM lane quadrant = warp % 4).
// Persistent CTAs loop over units (pose or pose pair); weights stay resident.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstdlib>
#include <cstring>
#include <vector>

#include "common.cuh"
#include "umma_conv.cuh"

namespace fs {
namespace umma {

// ---------------------------------------------------------------------------
// PTX wrappers
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void fence_barrier_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void tma_load_5d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1,
                                            int c2, int c3, int c4) {
  asm volatile(
      "cp.async.bulk.tensor.5d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5, %6, %7}], [%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(c4)
      : "memory");
}
__device__ __forceinline__ void tma_load_4d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1,
                                            int c2, int c3) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5, %6}], [%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
      : "memory");
}
__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// K-major, SWIZZLE_NONE UMMA shared-memory descriptor (sm_100 version 1).
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((saddr >> 4) & 0x3FFFu);
  d |= static_cast<uint64_t>((lbo >> 4) & 0x3FFFu) << 16;
  d |= static_cast<uint64_t>((sbo >> 4) & 0x3FFFu) << 32;
  d |= static_cast<uint64_t>(1) << 46;
  return d;
}
// kind::f16 instruction descriptor: BF16 x BF16 -> F32, both K-major.
__host__ __device__ constexpr uint32_t idesc_bf16(int M, int N) {
  return (1u << 4) | (1u << 7) | (1u << 10) | (static_cast<uint32_t>(N >> 3) << 17) |
         (static_cast<uint32_t>(M >> 4) << 24);
}
__device__ __forceinline__ void umma_bf16(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(d_tmem),
      "l"(a), "l"(b), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void umma_tf32(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(d_tmem),
      "l"(a), "l"(b), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float* v) {
  uint32_t r[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
        "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}

__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float* v) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}

__device__ __forceinline__ void tmem_zero16(uint32_t taddr) {
  const uint32_t z = 0;
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1};" ::"r"(taddr),
      "r"(z)
      : "memory");
}

__device__ __forceinline__ void tmem_zero32(uint32_t taddr) {
  const uint32_t z = 0;
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,"
      "%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1};" ::"r"(taddr), "r"(z)
      : "memory");
}

__host__ __device__ constexpr int align_to(int x, int a) { return (x + a - 1) / a * a; }
__host__ __device__ constexpr int pow2_cols(int x) {
  return x <= 32 ? 32 : x <= 64 ? 64 : x <= 128 ? 128 : x <= 256 ? 256 : 512;
}

// ---------------------------------------------------------------------------
// layer configuration
// ---------------------------------------------------------------------------
constexpr int kSlots = 8;   // TMEM accumulator slots (output planes in flight) per tile

// X3 (FS_PREC_MIXED): fp32-class 3-pass split on the same tensor cores.  An
// fp32 operand x = hi + lo with hi = bf16(x), lo = bf16(x - hi) (relative
// error ~2^-16); A.B ~ Alo.Bhi + Ahi.Blo + Ahi.Bhi, all accumulated in the
// same fp32 TMEM slot.  Activations travel as two bf16 tensors (hi, lo);
// weights hold a hi and a lo set.  AEX: the A operand is exact in bf16 (the
// voxel grid's integer counts), so its lo pass is skipped (2 passes).
template <int G_, int CIN_, int COUT_, int KS_, int POSES_, bool POOL_, bool RESID_, bool OUT_F32_, int NSPLIT_,
          int RING_ = 4, bool X3_ = false, bool AEX_ = false>
struct Cfg {
  static constexpr int G = G_, CIN = CIN_, COUT = COUT_, KS = KS_, POSES = POSES_, NSPLIT = NSPLIT_;
  static constexpr bool POOL = POOL_, RESID = RESID_, OUT_F32 = OUT_F32_, X3 = X3_, AEX = AEX_;
  static constexpr int W_SETS = X3 ? 2 : 1;                // weight sets: hi (+ lo)
  static constexpr int A_SETS = (X3 && !AEX) ? 2 : 1;      // staged input sets per plane: hi (+ lo)
  static constexpr int R = KS / 2;
  static constexpr int HP = G + 2 * R, WP = G + 2 * R;
  static constexpr int CHUNKS = CIN / 8;
  static constexpr int TILES = G / 8;                      // w halves per plane
  static_assert(G * POSES == 16, "M = 8 w x G h x POSES = 128");
  static constexpr int BOX_BYTES = HP * POSES * WP * 16;  // one TMA box (8 channels)
  static constexpr int CHUNK_BYTES = align_to(BOX_BYTES, 128);
  static constexpr int PLANE_BYTES = A_SETS * CHUNKS * CHUNK_BYTES;   // [set][chunk]
  static constexpr int RING = RING_;                       // staged input planes (each consumed once)
  static constexpr int NCTA = COUT / NSPLIT;               // output channels per CTA
  static constexpr int NG = NCTA / 8;
  static constexpr int STEPS_PER_PLANE = (CIN == 8) ? (KS * KS + 1) / 2 : KS * KS * (CIN / 16);
  static constexpr int KSTEPS = KS * STEPS_PER_PLANE;
  static constexpr int JSTEP = NG * 128;                   // bytes of one kernel plane's N rows (one K chunk)
  static constexpr int STEP_BYTES = 2 * KS * JSTEP;        // one (kh,kw,chunk) step: [kc][kd desc][cout]
  static constexpr int W_BYTES = STEPS_PER_PLANE * STEP_BYTES;   // per N slice and weight set
  static constexpr int SLOT_COLS = NCTA;
  static constexpr int TMEM_COLS = pow2_cols(TILES * kSlots * NCTA);
  static_assert(TILES * kSlots * NCTA <= 512, "TMEM budget");
  static_assert(G % kSlots == 0 && kSlots >= KS, "slot ring");
  static_assert(KS * NCTA <= 256 && NCTA % 16 == 0 && (NCTA % 32 == 0 || NCTA == 16), "stacked N");
  static constexpr int NPLANES = G + KS - 1;               // padded planes per unit
  static constexpr uint32_t SBO = WP * 16;
  static constexpr int RING_OFF = align_to(W_SETS * W_BYTES, 1024);
  static constexpr int BAR_OFF = RING_OFF + RING * PLANE_BYTES;
  // a 512-column TMEM allocation admits one CTA per SM: request enough shared
  // memory that the scheduler never co-locates two (the second would block
  // in tcgen05.alloc until the first, persistent one exits)
  static constexpr int SMEM = (TMEM_COLS == 512 && BAR_OFF + 256 < 116 * 1024) ? 116 * 1024 : BAR_OFF + 256;
  static_assert(SMEM <= 227 * 1024, "shared memory budget");
};

// conv1 8->32 k5 on 16^3; conv2 32->32 k3 +pool; conv3 32->64 k3 (pose pairs);
// conv4 64->64 k3 +residual +pool (pose pairs, N split over 2 CTAs).
using C1 = Cfg<16, 8, 32, 5, 1, false, false, false, 1, 6>;
// (ring depths leave room for one or two co-resident radius-graph CTAs of the
// overlapped graph branch: conv2 118.5 KB, conv4 162 KB)
using C2 = Cfg<16, 32, 32, 3, 1, true, false, false, 1, 3>;
using C3 = Cfg<8, 32, 64, 3, 2, false, false, false, 1, 4>;
using C4 = Cfg<8, 64, 64, 3, 2, true, true, true, 2, 2>;
// X3 chain (FS_PREC_MIXED): twice the weights and staged planes, so conv3/conv4
// split N over 2/4 CTAs and conv2/conv4 stage 2 planes ahead
using C1X = Cfg<16, 8, 32, 5, 1, false, false, false, 1, 6, true>;
using C2X = Cfg<16, 32, 32, 3, 1, true, false, false, 1, 2, true>;
using C3X = Cfg<8, 32, 64, 3, 2, false, false, false, 2, 4, true>;
using C4X = Cfg<8, 64, 64, 3, 2, true, true, true, 4, 2, true>;

// Per K-step A-descriptor low word (start-address and LBO fields, 16-byte
// units) relative to the plane base of the step's kd.
template <class L>
__host__ __device__ constexpr uint32_t a_step_lo(int s) {
  if constexpr (L::CIN == 8) {
    // two kernel offsets of the same kd plane per MMA (8 channels each)
    const int oa = 2 * s, ob = 2 * s + 1;
    const int kha = oa / L::KS, kwa = oa % L::KS;
    const int off = (kha * L::POSES * L::WP + kwa) * 16;
    // zero-weight dummy second chunk: LBO 0 re-reads chunk 0, which is finite
    // data (a past-the-plane read could hit mbarrier words whose bit patterns
    // are NaN, and 0*NaN = NaN)
    const int lbo = ob < L::KS * L::KS
                        ? ((ob / L::KS - kha) * L::POSES * L::WP + (ob % L::KS - kwa)) * 16 : 0;
    return static_cast<uint32_t>(off >> 4) | (static_cast<uint32_t>(lbo >> 4) << 16);
  } else {
    // one kernel offset, channel chunks (2cp, 2cp+1) per MMA (LBO = chunk stride)
    constexpr int CP = L::CIN / 16;
    const int cp = s % CP, o = s / CP;
    const int off = (2 * cp) * L::CHUNK_BYTES + ((o / L::KS) * L::POSES * L::WP + (o % L::KS)) * 16;
    return static_cast<uint32_t>(off >> 4);
  }
}

struct ConvParams {
  const char* w;            // packed B operands, NSPLIT slices of W_SETS x W_BYTES
  const float* bias;        // [COUT]
  const __nv_bfloat16* residual;   // [P][G^3][COUT] (conv4: h3; X3: its hi part)
  const __nv_bfloat16* residual_lo;   // X3: lo part of h3
  void* out;
  void* out_lo;             // X3, bf16 outputs: the lo part
  int n_poses;
};

// 8 fp32 values -> one 16-byte bf16 row at uint4 index i of `hi` (and, X3,
// their residuals x - bf16(x) rounded to bf16 at the same index of `lo`)
template <bool X3>
__device__ __forceinline__ void store_split8(void* hi, void* lo, size_t i, const float* x) {
  uint4 ph, pl;
  __nv_bfloat162* h2 = reinterpret_cast<__nv_bfloat162*>(&ph);
  __nv_bfloat162* l2 = reinterpret_cast<__nv_bfloat162*>(&pl);
#pragma unroll
  for (int t = 0; t < 4; ++t) {
    h2[t] = __floats2bfloat162_rn(x[2 * t], x[2 * t + 1]);
    if constexpr (X3) {
      const float2 hf = __bfloat1622float2(h2[t]);
      l2[t] = __floats2bfloat162_rn(x[2 * t] - hf.x, x[2 * t + 1] - hf.y);
    }
  }
  reinterpret_cast<uint4*>(hi)[i] = ph;
  if constexpr (X3) reinterpret_cast<uint4*>(lo)[i] = pl;
}

// ---------------------------------------------------------------------------
// the kernel
// ---------------------------------------------------------------------------
template <class L>
__global__ void __launch_bounds__(192, 1) conv_umma_kernel(const __grid_constant__ CUtensorMap tmap,
                                                           const __grid_constant__ CUtensorMap tmap_lo,
                                                           ConvParams prm) {
  extern __shared__ __align__(1024) unsigned char smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  unsigned char* wsm = smem;
  unsigned char* ring = smem + L::RING_OFF;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L::BAR_OFF);
  uint64_t* full = bars;                   // [RING]   plane staged
  uint64_t* empty = bars + L::RING;        // [RING]   plane's MMAs done
  uint64_t* tfull = bars + 2 * L::RING;    // [kSlots] output plane accumulated
  uint64_t* tempty = tfull + kSlots;       // [kSlots] slot drained and zeroed
  uint64_t* wbar = tempty + kSlots;        // [1]
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(wbar + 1);

  const int nsl = blockIdx.y;              // N slice
  const int n_units = (prm.n_poses + L::POSES - 1) / L::POSES;

  if (threadIdx.x == 0) {
    for (int i = 0; i < L::RING; ++i) { mbar_init(&full[i], 1); mbar_init(&empty[i], 1); }
    for (int i = 0; i < kSlots; ++i) { mbar_init(&tfull[i], 1); mbar_init(&tempty[i], 128); }
    mbar_init(wbar, 1);
    fence_barrier_init();
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_holder)),
                 "r"(L::TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_holder;

  if (warp == 0) {
    // ===================== TMA producer =====================
    if (lane == 0) {
      constexpr int WB = L::W_SETS * L::W_BYTES;
      const char* wsrc = prm.w + static_cast<size_t>(nsl) * WB;
      mbar_expect_tx(wbar, WB);
      for (int off = 0; off < WB; off += 32768) {
        const int n = min(32768, WB - off);
        bulk_load(wsm + off, wsrc + off, n, wbar);
      }
      uint32_t gq = 0;
      for (int u = blockIdx.x; u < n_units; u += gridDim.x) {
        const int p0 = u * L::POSES;
        // only the G real input planes are staged: the KS-1 "same"-padding
        // planes are all zero and contribute nothing (see the issuer)
        for (int q = L::R; q < L::G + L::R; ++q, ++gq) {
          const int slot = gq % L::RING;
          mbar_wait(&empty[slot], ((gq / L::RING) & 1) ^ 1);
          mbar_expect_tx(&full[slot], L::A_SETS * L::CHUNKS * L::BOX_BYTES);
          unsigned char* dst = ring + slot * L::PLANE_BYTES;
          for (int c = 0; c < L::CHUNKS; ++c)
            tma_load_5d(dst + c * L::CHUNK_BYTES, &tmap, &full[slot], -8 * L::R, p0, -L::R, q - L::R, c);
          if constexpr (L::A_SETS == 2)
            for (int c = 0; c < L::CHUNKS; ++c)
              tma_load_5d(dst + (L::CHUNKS + c) * L::CHUNK_BYTES, &tmap_lo, &full[slot], -8 * L::R, p0, -L::R,
                          q - L::R, c);
        }
      }
    }
  } else if (warp == 1) {
    // ===================== UMMA issuer =====================
    // The whole warp walks the schedule (descriptor math stays warp-uniform)
    // and lane 0 issues.  Input plane q: one stacked MMA per step and tile
    // (two where the output planes q-KS+1..q wrap around the slot ring).
    mbar_wait(wbar, 0);
    const uint32_t wbase = smem_u32(wsm);
    const uint32_t rbase = smem_u32(ring);
    constexpr uint32_t A_HI = ((L::SBO >> 4) & 0x3FFFu) | (1u << 14);
    constexpr uint32_t B_HI = (128u >> 4) | (1u << 14);
    constexpr uint32_t A_LBO = (L::CIN == 8) ? 0u : ((static_cast<uint32_t>(L::CHUNK_BYTES) >> 4) << 16);
    constexpr uint32_t B_STEP = L::STEP_BYTES >> 4;
    constexpr uint32_t B_J = L::JSTEP >> 4;
    const uint32_t b_lo0 = ((wbase >> 4) & 0x3FFFu) | (((L::KS * L::JSTEP) >> 4) << 16);
    uint32_t gq = 0, uo = 0;
    for (int u = blockIdx.x; u < n_units; u += gridDim.x, uo += L::G) {
      for (int q = 0; q < L::NPLANES; ++q) {
        // input planes q < R and q >= G + R are the zero "same" padding: their
        // MMAs would add exact zeros, so they are skipped (no staging, no MMA;
        // output slots start zeroed) -- 20% of the MMAs at KS = 5 / G = 8
        const bool real = q >= L::R && q < L::G + L::R;
        const uint32_t rs = gq % L::RING;
        if (real) mbar_wait(&full[rs], (gq / L::RING) & 1);
        const int dlo = q - L::KS + 1 > 0 ? q - L::KS + 1 : 0;
        const int dhi = q < L::G - 1 ? q : L::G - 1;
        if (q < L::G) {   // output plane q enters: its slot must be drained and zeroed
          const uint32_t o = uo + q;
          mbar_wait(&tempty[o % kSlots], (o / kSlots) & 1);
        }
        tc_fence_after();
        if (real) {
        // [dlo, dhi] split where it crosses a multiple of kSlots (G % kSlots == 0,
        // so output d of every unit lives in slot d % kSlots)
        const int dmid = (dlo / kSlots + 1) * kSlots;      // first plane of the next slot cycle
        const int nseg = dhi >= dmid ? 2 : 1;
        const uint32_t pbase = rbase + rs * L::PLANE_BYTES;
#pragma unroll 1
        for (int sg = 0; sg < nseg; ++sg) {
          const int a = sg == 0 ? dlo : dmid;
          const int b = sg == 0 ? (nseg == 2 ? dmid - 1 : dhi) : dhi;
          const uint32_t idesc = idesc_bf16(128, (b - a + 1) * L::NCTA);
          const uint32_t j0 = static_cast<uint32_t>(L::KS - 1 - q + a);   // kd = q - a, stored descending
#pragma unroll
          for (int wh = 0; wh < L::TILES; ++wh) {
            const uint32_t dtm = tmem_base + (wh * kSlots + (a % kSlots)) * L::SLOT_COLS;
            const uint32_t a_lo0 = (((pbase + wh * 128u) >> 4) & 0x3FFFu) | A_LBO;
            const uint32_t b_lo1 = b_lo0 + j0 * B_J;
#pragma unroll
            for (int s2 = 0; s2 < L::STEPS_PER_PLANE; ++s2) {
              const uint32_t a_lo = a_lo0 + a_step_lo<L>(s2);
              const uint32_t b_lo = b_lo1 + s2 * B_STEP;
              if (lane == 0) {
                if constexpr (L::X3) {
                  // small cross terms first, the hi.hi product last (one fp32 slot)
                  constexpr uint32_t A_SET = (L::CHUNKS * L::CHUNK_BYTES) >> 4;
                  constexpr uint32_t B_SET = L::W_BYTES >> 4;
                  if constexpr (L::A_SETS == 2)
                    umma_bf16(dtm, (static_cast<uint64_t>(A_HI) << 32) | (a_lo + A_SET),
                              (static_cast<uint64_t>(B_HI) << 32) | b_lo, idesc, 1u);
                  umma_bf16(dtm, (static_cast<uint64_t>(A_HI) << 32) | a_lo,
                            (static_cast<uint64_t>(B_HI) << 32) | (b_lo + B_SET), idesc, 1u);
                }
                umma_bf16(dtm, (static_cast<uint64_t>(A_HI) << 32) | a_lo,
                          (static_cast<uint64_t>(B_HI) << 32) | b_lo, idesc, 1u);
              }
            }
          }
        }
        if (lane == 0) umma_commit(&empty[rs]);         // plane q is read by no later MMA
        ++gq;
        }   // real
        if (lane == 0 && q >= L::KS - 1) {               // output plane q-KS+1 is complete
          const uint32_t o = uo + q - L::KS + 1;
          umma_commit(&tfull[o % kSlots]);
        }
        __syncwarp();
      }
    }
  } else {
    // ===================== epilogue (warps 2..5) =====================
    const int quad = warp & 3;
    const int r = quad * 32 + lane;                 // tile row == TMEM lane
    const int grp = r >> 3, wl = r & 7;
    const int h = grp / L::POSES, ps = grp % L::POSES;
    const int n0 = nsl * L::NCTA;
    const uint32_t tq = tmem_base + (static_cast<uint32_t>(quad * 32) << 16);
    // every slot starts zeroed (MMAs always accumulate)
#pragma unroll 1
    for (int s = 0; s < kSlots; ++s)
#pragma unroll
      for (int wh = 0; wh < L::TILES; ++wh)
#pragma unroll
        for (int c0 = 0; c0 < L::NCTA; c0 += 32) {
          if constexpr (L::NCTA % 32 == 0) tmem_zero32(tq + (wh * kSlots + s) * L::SLOT_COLS + c0);
          else tmem_zero16(tq + (wh * kSlots + s) * L::SLOT_COLS + c0);   // NCTA == 16 (C4X)
        }
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    tc_fence_before();
    for (int s = 0; s < kSlots; ++s) mbar_arrive(&tempty[s]);
    float bias[L::NCTA];
#pragma unroll
    for (int j = 0; j < L::NCTA; ++j) bias[j] = prm.bias[n0 + j];
    float pmax[L::POOL ? L::TILES * L::NCTA : 1];
    uint32_t o = 0;
    for (int u = blockIdx.x; u < n_units; u += gridDim.x) {
      const int pose = u * L::POSES + ps;
      const bool live = pose < prm.n_poses;
      for (int d = 0; d < L::G; ++d, ++o) {
        const int slot = o % kSlots;
        mbar_wait(&tfull[slot], (o / kSlots) & 1);
        tc_fence_after();
#pragma unroll
        for (int wh = 0; wh < L::TILES; ++wh) {
          const int w = wh * 8 + wl;
          float v[L::NCTA];
#pragma unroll
          for (int c0 = 0; c0 < L::NCTA; c0 += 32) {
            const uint32_t ta = tq + (wh * kSlots + slot) * L::SLOT_COLS + c0;
            if constexpr (L::NCTA % 32 == 0) {
              tmem_ld32(ta, v + c0);
              tmem_zero32(ta);
            } else {
              tmem_ld16(ta, v + c0);
              tmem_zero16(ta);
            }
          }
#pragma unroll
          for (int j = 0; j < L::NCTA; ++j) v[j] = fmaxf(v[j] + bias[j], 0.0f);
          // chunk-major activations: [pose][C/8][d][h][w][8]
          constexpr size_t G3 = static_cast<size_t>(L::G) * L::G * L::G;
          const size_t vox = (static_cast<size_t>(d) * L::G + h) * L::G + w;
          if constexpr (L::RESID) {
            if (live) {
              const uint4* rp = reinterpret_cast<const uint4*>(prm.residual) +
                                (static_cast<size_t>(pose) * (L::COUT / 8) + n0 / 8) * G3 + vox;
#pragma unroll
              for (int q = 0; q < L::NCTA / 8; ++q) {
                uint4 pk = rp[q * G3];
                const __nv_bfloat162* b2 = reinterpret_cast<const __nv_bfloat162*>(&pk);
                float2 rl[4] = {};
                if constexpr (L::X3) {   // h3 = hi + lo
                  const uint4 pl = reinterpret_cast<const uint4*>(prm.residual_lo)[(rp - reinterpret_cast<const uint4*>(prm.residual)) + q * G3];
                  const __nv_bfloat162* l2 = reinterpret_cast<const __nv_bfloat162*>(&pl);
#pragma unroll
                  for (int t = 0; t < 4; ++t) rl[t] = __bfloat1622float2(l2[t]);
                }
#pragma unroll
                for (int t = 0; t < 4; ++t) {
                  float2 f = __bfloat1622float2(b2[t]);
                  v[q * 8 + 2 * t] += f.x + rl[t].x;
                  v[q * 8 + 2 * t + 1] += f.y + rl[t].y;
                }
              }
            }
          }
          if constexpr (L::POOL) {
            constexpr int HX = 8 * L::POSES;        // lane distance of the h partner
#pragma unroll
            for (int j = 0; j < L::NCTA; ++j) {
              float x = v[j];
              x = fmaxf(x, __shfl_xor_sync(0xffffffffu, x, 1));
              x = fmaxf(x, __shfl_xor_sync(0xffffffffu, x, HX));
              if (d & 1) x = fmaxf(x, pmax[wh * L::NCTA + j]);
              pmax[wh * L::NCTA + j] = x;
            }
            if ((d & 1) && live && !(wl & 1) && !(h & 1)) {
              constexpr int GO = L::G / 2;
              if constexpr (L::OUT_F32) {
                // final layer: NDHWC float32 (the dense1 flatten order)
                const size_t ov = ((static_cast<size_t>(pose) * GO + d / 2) * GO + h / 2) * GO + w / 2;
                float4* op = reinterpret_cast<float4*>(reinterpret_cast<float*>(prm.out) + ov * L::COUT + n0);
#pragma unroll
                for (int q = 0; q < L::NCTA / 4; ++q)
                  op[q] = make_float4(pmax[wh * L::NCTA + 4 * q], pmax[wh * L::NCTA + 4 * q + 1],
                                      pmax[wh * L::NCTA + 4 * q + 2], pmax[wh * L::NCTA + 4 * q + 3]);
              } else {
                constexpr size_t GO3 = static_cast<size_t>(GO) * GO * GO;
                const size_t ovx = (static_cast<size_t>(d / 2) * GO + h / 2) * GO + w / 2;
                const size_t oi = (static_cast<size_t>(pose) * (L::COUT / 8) + n0 / 8) * GO3 + ovx;
#pragma unroll
                for (int q = 0; q < L::NCTA / 8; ++q)
                  store_split8<L::X3>(prm.out, prm.out_lo, oi + q * GO3, pmax + wh * L::NCTA + q * 8);
              }
            }
          } else if (live) {
            const size_t oi = (static_cast<size_t>(pose) * (L::COUT / 8) + n0 / 8) * G3 + vox;
#pragma unroll
            for (int q = 0; q < L::NCTA / 8; ++q) store_split8<L::X3>(prm.out, prm.out_lo, oi + q * G3, v + q * 8);
          }
        }
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        tc_fence_before();
        mbar_arrive(&tempty[slot]);
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(L::TMEM_COLS));
  }
}

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------
static PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

// 5-D map over a chunk-major bf16 activation [P][C/8][G][G][G][8] with
// dimension order ((w,c8), pose, h, d, chunk): the innermost box row is a
// whole padded w-row of one chunk (WP*16 bytes, not 16), and putting pose
// between (w,c8) and h makes one box fill the (h, pose, w) interleave.
template <class L>
static int make_map(CUtensorMap* map, const void* base, int n_poses) {
  auto fn = encode_fn();
  if (!fn) return FS_ECUDA;
  const cuuint64_t G = L::G, CH = L::CIN / 8;
  cuuint64_t dims[5] = {G * 8, static_cast<cuuint64_t>(n_poses), G, G, CH};
  cuuint64_t strides[4] = {CH * G * G * G * 16, G * 16, G * G * 16, G * G * G * 16};
  cuuint32_t box[5] = {static_cast<cuuint32_t>(L::WP * 8), static_cast<cuuint32_t>(L::POSES),
                       static_cast<cuuint32_t>(L::HP), 1, 1};
  cuuint32_t estr[5] = {1, 1, 1, 1, 1};
  CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 5, const_cast<void*>(base), dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? FS_OK : FS_ECUDA;
}

static int g_num_sms = 0;

template <class L>
static int launch_layer(const void* in, ConvParams prm, cudaStream_t st, const void* in_lo = nullptr) {
  if (prm.n_poses <= 0) return FS_OK;
  CUtensorMap map, map_lo;
  int rc = make_map<L>(&map, in, prm.n_poses);
  if (rc) return rc;
  if (L::A_SETS == 2 && !in_lo) return FS_EINVAL;
  if ((rc = make_map<L>(&map_lo, L::A_SETS == 2 ? in_lo : in, prm.n_poses))) return rc;
  if (!g_num_sms) {
    int dev = 0;
    FS_CUDA_CHECK(cudaGetDevice(&dev));
    FS_CUDA_CHECK(cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev));
  }
  FS_CUDA_CHECK(cudaFuncSetAttribute(conv_umma_kernel<L>, cudaFuncAttributeMaxDynamicSharedMemorySize, L::SMEM));
  const int units = (prm.n_poses + L::POSES - 1) / L::POSES;
  static const bool one_per_sm = getenv("FS_UMMA_ONE_CTA_PER_SM") != nullptr;
  const int per_sm = (!one_per_sm && L::TMEM_COLS <= 256 && (227 * 1024) / (L::SMEM + 1024) >= 2) ? 2 : 1;
  // FS_CONV_SMS (A/B): cap the persistent grid below the SM count, leaving
  // SMs to a concurrently running graph branch
  static const int conv_sms = getenv("FS_CONV_SMS") ? atoi(getenv("FS_CONV_SMS")) : 0;
  const int sms = conv_sms > 0 && conv_sms < g_num_sms ? conv_sms : g_num_sms;
  const int ctas = max(1, min(units, sms * per_sm / L::NSPLIT));
  dim3 grid(ctas, L::NSPLIT);
  conv_umma_kernel<L><<<grid, 192, L::SMEM, st>>>(map, map_lo, prm);
  FS_LAUNCH_CHECK();
  return FS_OK;
}

// ---------------------------------------------------------------------------
// dense1 of the voxel head on tcgen05 (kind::tf32):
//   y[P][128] = relu(x[P][K] . W + b)      (models.py:316-318, autodiff.py:161-173)
// x = the pooled conv4 output (fp32, NDHWC flatten order, rows padded to a
// multiple of 128), wt = W^T fp32 [128][K] in the same K order.  One CTA per
// 128-pose tile: TMA streams 32-wide K slabs of x and W^T (4-D tensor maps
// whose boxes land in the K-major no-swizzle core-matrix layout: 8 rows x
// 16 B, K chunks 128 B apart, 8-row groups 1 KB apart) through a 4-stage
// ring; one thread issues M=128 N=128 K=8 MMAs into a 128-column TMEM
// accumulator; 4 epilogue warps add the bias and apply ReLU.  The operands
// are rounded to tf32 by the tensor core (10-bit mantissa; fp32 accumulate).
// ---------------------------------------------------------------------------
namespace dn {
constexpr int BM = 128, BN = 128, BK = 32, STAGES = 4;
constexpr int A_BYTES = BM * BK * 4, B_BYTES = BN * BK * 4, STAGE_BYTES = A_BYTES + B_BYTES;
constexpr int BAR_OFF = STAGES * STAGE_BYTES;
constexpr int SMEM = BAR_OFF + 256;
constexpr uint32_t IDESC = (1u << 4) | (2u << 7) | (2u << 10) | (static_cast<uint32_t>(BN >> 3) << 17) |
                           (static_cast<uint32_t>(BM >> 4) << 24);
}  // namespace dn

__global__ void __launch_bounds__(192, 1) dense_tf32_kernel(const __grid_constant__ CUtensorMap ta,
                                                            const __grid_constant__ CUtensorMap tb,
                                                            const float* __restrict__ bias, float* __restrict__ y,
                                                            int P, int K) {
  extern __shared__ __align__(1024) unsigned char smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + dn::BAR_OFF);
  uint64_t* full = bars;
  uint64_t* empty = bars + dn::STAGES;
  uint64_t* done = bars + 2 * dn::STAGES;
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(done + 1);
  const int nk = K / dn::BK;
  if (threadIdx.x == 0) {
    for (int i = 0; i < dn::STAGES; ++i) { mbar_init(&full[i], 1); mbar_init(&empty[i], 1); }
    mbar_init(done, 1);
    fence_barrier_init();
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_holder)),
                 "r"(dn::BN));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_holder;
  if (warp == 0) {
    if (lane == 0) {
      for (int kb = 0; kb < nk; ++kb) {
        const int sl = kb % dn::STAGES;
        mbar_wait(&empty[sl], ((kb / dn::STAGES) & 1) ^ 1);
        mbar_expect_tx(&full[sl], dn::STAGE_BYTES);
        unsigned char* st = smem + sl * dn::STAGE_BYTES;
        tma_load_4d(st, &ta, &full[sl], 0, 0, kb * (dn::BK / 4), blockIdx.x * (dn::BM / 8));
        tma_load_4d(st + dn::A_BYTES, &tb, &full[sl], 0, 0, kb * (dn::BK / 4), 0);
      }
    }
  } else if (warp == 1) {
    const uint32_t base = smem_u32(smem);
    for (int kb = 0; kb < nk; ++kb) {
      const int sl = kb % dn::STAGES;
      mbar_wait(&full[sl], (kb / dn::STAGES) & 1);
      tc_fence_after();
      const uint32_t a0 = base + sl * dn::STAGE_BYTES, b0 = a0 + dn::A_BYTES;
#pragma unroll
      for (int kk = 0; kk < dn::BK / 8; ++kk)   // K = 8 per MMA: two 16-byte chunks, 128 B apart
        if (lane == 0)
          umma_tf32(tmem, sdesc(a0 + kk * 256, 128, 1024), sdesc(b0 + kk * 256, 128, 1024), dn::IDESC,
                    (kb | kk) != 0 ? 1u : 0u);
      if (lane == 0) umma_commit(&empty[sl]);
      __syncwarp();
    }
    if (lane == 0) umma_commit(done);
    __syncwarp();
  } else {
    const int quad = warp & 3;
    const int row = blockIdx.x * dn::BM + quad * 32 + lane;
    mbar_wait(done, 0);
    tc_fence_after();
#pragma unroll
    for (int c0 = 0; c0 < dn::BN; c0 += 32) {
      float v[32];
      tmem_ld32(tmem + (static_cast<uint32_t>(quad * 32) << 16) + c0, v);
      if (row < P) {
        float4* o = reinterpret_cast<float4*>(y + static_cast<size_t>(row) * dn::BN + c0);
#pragma unroll
        for (int q = 0; q < 8; ++q)
          o[q] = make_float4(fmaxf(v[4 * q] + bias[c0 + 4 * q], 0.f), fmaxf(v[4 * q + 1] + bias[c0 + 4 * q + 1], 0.f),
                             fmaxf(v[4 * q + 2] + bias[c0 + 4 * q + 2], 0.f),
                             fmaxf(v[4 * q + 3] + bias[c0 + 4 * q + 3], 0.f));
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(dn::BN));
  }
}

// fp32 [rows][K] (row stride K) as (4 elems, 8 rows, K/4 chunks, rows/8 groups)
static int make_dense_map(CUtensorMap* map, const void* base, int rows, int K) {
  auto fn = encode_fn();
  if (!fn) return FS_ECUDA;
  cuuint64_t dims[4] = {4, 8, static_cast<cuuint64_t>(K / 4), static_cast<cuuint64_t>((rows + 7) / 8)};
  cuuint64_t strides[3] = {static_cast<cuuint64_t>(K) * 4, 16, static_cast<cuuint64_t>(K) * 4 * 8};
  cuuint32_t box[4] = {4, 8, dn::BK / 4, 16};
  cuuint32_t estr[4] = {1, 1, 1, 1};
  CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, const_cast<void*>(base), dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? FS_OK : FS_ECUDA;
}

bool dense_tf32_ok(int K, int N) { return N == dn::BN && K % dn::BK == 0 && K >= dn::BK; }

size_t dense_rows_padded(int64_t P) { return static_cast<size_t>((P + dn::BM - 1) / dn::BM * dn::BM); }

int dense_tf32(const float* x, int P, int K, const float* wt, int N, const float* bias, float* y, cudaStream_t st) {
  if (P <= 0) return FS_OK;
  if (!dense_tf32_ok(K, N)) return FS_ENOTSUP;
  CUtensorMap ta, tb;
  int rc = make_dense_map(&ta, x, static_cast<int>(dense_rows_padded(P)), K);
  if (rc) return rc;
  if ((rc = make_dense_map(&tb, wt, N, K))) return rc;
  FS_CUDA_CHECK(cudaFuncSetAttribute(dense_tf32_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, dn::SMEM));
  dense_tf32_kernel<<<(P + dn::BM - 1) / dn::BM, 192, dn::SMEM, st>>>(ta, tb, bias, y, P, K);
  FS_LAUNCH_CHECK();
  return FS_OK;
}

bool supports(const fs_model_desc& d) {
  return d.grid_extent == 16 && d.in_channels == 8 && d.conv_filters_1 == 32 && d.conv_filters_2 == 64 &&
         d.kernel_1 == 5 && d.kernel_2 == 3 && !d.residual_1 && d.residual_2 && !d.batch_norm;
}

static constexpr size_t OFF_W1 = 0;
static constexpr size_t OFF_W2 = align_to(C1::W_BYTES * C1::NSPLIT, 1024);
static constexpr size_t OFF_W3 = OFF_W2 + align_to(C2::W_BYTES * C2::NSPLIT, 1024);
static constexpr size_t OFF_W4 = OFF_W3 + align_to(C3::W_BYTES * C3::NSPLIT, 1024);
static constexpr size_t OFF_X1 = OFF_W4 + align_to(C4::W_BYTES * C4::NSPLIT, 1024);
static constexpr size_t OFF_X2 = OFF_X1 + align_to(2 * C1X::W_BYTES * C1X::NSPLIT, 1024);
static constexpr size_t OFF_X3 = OFF_X2 + align_to(2 * C2X::W_BYTES * C2X::NSPLIT, 1024);
static constexpr size_t OFF_X4 = OFF_X3 + align_to(2 * C3X::W_BYTES * C3X::NSPLIT, 1024);
static constexpr size_t W_TOTAL = OFF_X4 + align_to(2 * C4X::W_BYTES * C4X::NSPLIT, 1024);

size_t weights_bytes(const fs_model_desc& d) { return supports(d) ? W_TOTAL : 0; }

static uint16_t to_bf16(double x) {
  float f = static_cast<float>(x);
  uint32_t u;
  std::memcpy(&u, &f, 4);
  if ((u & 0x7f800000u) == 0x7f800000u) return static_cast<uint16_t>(u >> 16);   // inf/nan
  u += 0x7fffu + ((u >> 16) & 1u);                                                  // RNE
  return static_cast<uint16_t>(u >> 16);
}
static double from_bf16(uint16_t h) {
  const uint32_t u = static_cast<uint32_t>(h) << 16;
  float f;
  std::memcpy(&f, &u, 4);
  return f;
}
// the X3 lo part of a weight: bf16(w - bf16(w)), from the fp64 reference value
static uint16_t to_bf16_lo(double x) { return to_bf16(x - from_bf16(to_bf16(x))); }

// B operand layout per N slice: [step (kh,kw,chunk)][kchunk 2][kd descending]
// [n-group][8 rows][8 ch] bf16 -- the N rows of one step are the KS kernel
// planes side by side, so a stacked MMA over output planes a..b of input
// plane q reads the contiguous rows of kd = q-a down to q-b.
template <class L>
static void pack_layer(const double* w, char* out) {
  // w: reference [O][C][k][k][k]; per N slice: W_SETS sets of W_BYTES (hi, lo)
  const int K = L::KS, C = L::CIN;
  for (int sl = 0; sl < L::NSPLIT; ++sl)
  for (int set = 0; set < L::W_SETS; ++set) {
    uint16_t* o = reinterpret_cast<uint16_t*>(out + static_cast<size_t>(sl * L::W_SETS + set) * L::W_BYTES);
    std::memset(o, 0, L::W_BYTES);
    for (int s = 0; s < L::STEPS_PER_PLANE; ++s)
      for (int kc = 0; kc < 2; ++kc) {
        int kh, kw, c0;
        if constexpr (L::CIN == 8) {
          const int off = 2 * s + kc;
          if (off >= K * K) continue;     // zero-weight dummy chunk
          kh = off / K; kw = off % K; c0 = 0;
        } else {
          constexpr int CP = L::CIN / 16;
          const int cp = s % CP, off = s / CP;
          kh = off / K; kw = off % K; c0 = 16 * cp + 8 * kc;
        }
        for (int j = 0; j < K; ++j) {
          const int kd = K - 1 - j;
          for (int n = 0; n < L::NCTA; ++n) {
            const int oc = sl * L::NCTA + n;
            const size_t core = ((static_cast<size_t>(s) * 2 + kc) * K + j) * L::NG + n / 8;
            for (int e = 0; e < 8; ++e) {
              const int ic = c0 + e;
              const double v = w[((((size_t)oc * C + ic) * K + kd) * K + kh) * K + kw];
              o[core * 64 + (n % 8) * 8 + e] = set == 0 ? to_bf16(v) : to_bf16_lo(v);
            }
          }
        }
      }
  }
}

void pack_weights(const fs_model_desc& d, const double* c1, const double* c2, const double* c3, const double* c4,
                  char* out) {
  if (!supports(d) || !c1 || !c2 || !c3 || !c4) return;
  pack_layer<C1>(c1, out + OFF_W1);
  pack_layer<C2>(c2, out + OFF_W2);
  pack_layer<C3>(c3, out + OFF_W3);
  pack_layer<C4>(c4, out + OFF_W4);
  pack_layer<C1X>(c1, out + OFF_X1);
  pack_layer<C2X>(c2, out + OFF_X2);
  pack_layer<C3X>(c3, out + OFF_X3);
  pack_layer<C4X>(c4, out + OFF_X4);
}

// act1 [P][16^3][32] bf16, act2 (pooled) [P][8^3][32] bf16, act3 [P][8^3][64] bf16
static size_t act1_bytes(int64_t P) { return static_cast<size_t>(P) * 4096 * 32 * 2; }
static size_t act2_bytes(int64_t P) { return static_cast<size_t>(P + 1) * 512 * 32 * 2; }
static size_t act3_bytes(int64_t P) { return static_cast<size_t>(P + 1) * 512 * 64 * 2; }

size_t workspace_bytes(const fs_model_desc& d, int64_t P, bool x3) {
  if (!supports(d)) return 0;
  return (x3 ? 2 : 1) * (act1_bytes(P) + act2_bytes(P) + act3_bytes(P)) + 4096;
}

// X3 chain (FS_PREC_MIXED): activations as hi/lo bf16 pairs, 3-pass MMAs
int voxel_convs_x3(const fs_model_desc& d, const char* wblob, const float* b1, const float* b2, const float* b3,
                   const float* b4, int P, const __nv_bfloat16* grid, const __nv_bfloat16* grid_lo, char* ws,
                   float* flat_out, cudaStream_t st) {
  if (!supports(d)) return FS_ENOTSUP;
  if (P <= 0) return FS_OK;
  char* a1 = reinterpret_cast<char*>((reinterpret_cast<uintptr_t>(ws) + 1023) & ~static_cast<uintptr_t>(1023));
  char* a2 = a1 + act1_bytes(P);
  char* a3 = a2 + act2_bytes(P);
  char* l1 = a3 + act3_bytes(P);
  char* l2 = l1 + act1_bytes(P);
  char* l3 = l2 + act2_bytes(P);
  int rc;
  ConvParams p{};
  p.n_poses = P;
  mark_stage(ST_CONV1, st);
  p.w = wblob + OFF_X1; p.bias = b1; p.out = a1; p.out_lo = l1;
  if ((rc = launch_layer<C1X>(grid, p, st, grid_lo))) return rc;
  mark_stage(ST_CONV2, st);
  p.w = wblob + OFF_X2; p.bias = b2; p.out = a2; p.out_lo = l2;
  if ((rc = launch_layer<C2X>(a1, p, st, l1))) return rc;
  mark_stage(ST_CONV3, st);
  p.w = wblob + OFF_X3; p.bias = b3; p.out = a3; p.out_lo = l3;
  if ((rc = launch_layer<C3X>(a2, p, st, l2))) return rc;
  mark_stage(ST_CONV4, st);
  p.w = wblob + OFF_X4; p.bias = b4; p.out = flat_out; p.out_lo = nullptr;
  p.residual = reinterpret_cast<const __nv_bfloat16*>(a3); p.residual_lo = reinterpret_cast<const __nv_bfloat16*>(l3);
  return launch_layer<C4X>(a3, p, st, l3);
}

int voxel_convs(const fs_model_desc& d, const char* wblob, const float* b1, const float* b2, const float* b3,
                const float* b4, int P, const __nv_bfloat16* grid, char* ws, float* flat_out, cudaStream_t st) {
  if (!supports(d)) return FS_ENOTSUP;
  if (P <= 0) return FS_OK;
  char* a1 = reinterpret_cast<char*>((reinterpret_cast<uintptr_t>(ws) + 1023) & ~static_cast<uintptr_t>(1023));
  char* a2 = a1 + act1_bytes(P);
  char* a3 = a2 + act2_bytes(P);
  int rc;
  ConvParams p{};
  p.n_poses = P;
  mark_stage(ST_CONV1, st);
  p.w = wblob + OFF_W1; p.bias = b1; p.out = a1;
  if ((rc = launch_layer<C1>(grid, p, st))) return rc;
  mark_stage(ST_CONV2, st);
  p.w = wblob + OFF_W2; p.bias = b2; p.out = a2;
  if ((rc = launch_layer<C2>(a1, p, st))) return rc;
  mark_stage(ST_CONV3, st);
  p.w = wblob + OFF_W3; p.bias = b3; p.out = a3;
  if ((rc = launch_layer<C3>(a2, p, st))) return rc;
  mark_stage(ST_CONV4, st);
  p.w = wblob + OFF_W4; p.bias = b4; p.out = flat_out; p.residual = reinterpret_cast<const __nv_bfloat16*>(a3);
  if ((rc = launch_layer<C4>(a3, p, st))) return rc;
  return FS_OK;
}

__nv_bfloat16* act1_ptr(char* ws) {
  return reinterpret_cast<__nv_bfloat16*>((reinterpret_cast<uintptr_t>(ws) + 1023) & ~static_cast<uintptr_t>(1023));
}

// conv2..conv4 from an act1 produced elsewhere (the pocket-factored conv1)
int voxel_convs_from2(const fs_model_desc& d, const char* wblob, const float* b2, const float* b3, const float* b4,
                      int P, char* ws, float* flat_out, cudaStream_t st) {
  if (!supports(d)) return FS_ENOTSUP;
  if (P <= 0) return FS_OK;
  char* a1 = reinterpret_cast<char*>(act1_ptr(ws));
  char* a2 = a1 + act1_bytes(P);
  char* a3 = a2 + act2_bytes(P);
  int rc;
  ConvParams p{};
  p.n_poses = P;
  mark_stage(ST_CONV2, st);
  p.w = wblob + OFF_W2; p.bias = b2; p.out = a2;
  if ((rc = launch_layer<C2>(a1, p, st))) return rc;
  mark_stage(ST_CONV3, st);
  p.w = wblob + OFF_W3; p.bias = b3; p.out = a3;
  if ((rc = launch_layer<C3>(a2, p, st))) return rc;
  mark_stage(ST_CONV4, st);
  p.w = wblob + OFF_W4; p.bias = b4; p.out = flat_out; p.residual = reinterpret_cast<const __nv_bfloat16*>(a3);
  return launch_layer<C4>(a3, p, st);
}

// X3 workspace: a1, a2, a3 (hi) then l1, l2, l3 (lo)
__nv_bfloat16* act1_lo_ptr(char* ws, int64_t P) {
  return reinterpret_cast<__nv_bfloat16*>(reinterpret_cast<char*>(act1_ptr(ws)) + act1_bytes(P) + act2_bytes(P) +
                                          act3_bytes(P));
}

int voxel_convs_from2_x3(const fs_model_desc& d, const char* wblob, const float* b2, const float* b3, const float* b4,
                         int P, char* ws, float* flat_out, cudaStream_t st) {
  if (!supports(d)) return FS_ENOTSUP;
  if (P <= 0) return FS_OK;
  char* a1 = reinterpret_cast<char*>(act1_ptr(ws));
  char* a2 = a1 + act1_bytes(P);
  char* a3 = a2 + act2_bytes(P);
  char* l1 = a3 + act3_bytes(P);
  char* l2 = l1 + act1_bytes(P);
  char* l3 = l2 + act2_bytes(P);
  int rc;
  ConvParams p{};
  p.n_poses = P;
  mark_stage(ST_CONV2, st);
  p.w = wblob + OFF_X2; p.bias = b2; p.out = a2; p.out_lo = l2;
  if ((rc = launch_layer<C2X>(a1, p, st, l1))) return rc;
  mark_stage(ST_CONV3, st);
  p.w = wblob + OFF_X3; p.bias = b3; p.out = a3; p.out_lo = l3;
  if ((rc = launch_layer<C3X>(a2, p, st, l2))) return rc;
  mark_stage(ST_CONV4, st);
  p.w = wblob + OFF_X4; p.bias = b4; p.out = flat_out; p.out_lo = nullptr;
  p.residual = reinterpret_cast<const __nv_bfloat16*>(a3); p.residual_lo = reinterpret_cast<const __nv_bfloat16*>(l3);
  return launch_layer<C4X>(a3, p, st, l3);
}

int debug_layer(const fs_model_desc& d, const char* wblob, const float* bias, const float* residual_unused,
                int layer, int P, const void* in, const void* residual, void* out, cudaStream_t st) {
  (void)residual_unused;
  if (!supports(d)) return FS_ENOTSUP;
  ConvParams p{};
  p.n_poses = P; p.bias = bias; p.out = out;
  p.residual = reinterpret_cast<const __nv_bfloat16*>(residual);
  switch (layer) {
    case 1: p.w = wblob + OFF_W1; return launch_layer<C1>(in, p, st);
    case 2: p.w = wblob + OFF_W2; return launch_layer<C2>(in, p, st);
    case 3: p.w = wblob + OFF_W3; return launch_layer<C3>(in, p, st);
    case 4: p.w = wblob + OFF_W4; return launch_layer<C4>(in, p, st);
    default: return FS_EINVAL;
  }
}

}  // namespace umma
}  // namespace fs
