// tcgen05 implicit-GEMM engine v2 for conv forward / data-gradient (3xTF32).
//
// Why a second engine: in v1 both operands are gathered, split and stored to
// shared memory by producer warps; ncu (profiles/r01_conv2_fwd_v1.md) shows
// it issue-bound (IPC 1.5, tensor pipe 16%) and 3xTF32 needs
// 2x operand writes + 3x operand reads of shared memory per k-step.  v2:
//
//  * A (the pixel-major im2col operand, gathered from NCHW) never touches
//    shared memory: each producer thread owns one TMEM lane (= one output
//    pixel), gathers its K slice, splits it into TF32 big/small in registers
//    and writes both with tcgen05.st; the MMA reads A from TMEM
//    (tcgen05.mma ... [a_tmem], b_desc).
//  * B (the weights) is split and laid out ONCE per operator by a pack kernel
//    into the exact 128B-swizzled K-major shared-memory image, per (n-tile,
//    k-block); the GEMM fetches each stage with one cp.async.bulk (TMA) that
//    completes on the stage's mbarrier.  Shared memory then carries only the
//    B tile (1 write, 3 tensor-core reads per k-step).
//  * N tile = the whole output-channel extent up to 256 (rounded to 32), so
//    A is gathered once per output pixel tile.
//
// TMEM map (512 columns): nacc fp32 accumulators of BN columns at BN*b, then
// the A ring from abase = 64-aligned end of the accumulators: stage s holds
// A_big in [abase + 64*s, +32) and A_small in [abase + 64*s + 32, +32).  The
// ring is as deep as the columns allow (4..7 stages): a stage is recycled only
// after its MMAs complete and the commit reaches the producers (~2000 cycles),
// so narrow tiles (BN <= 64, 384 tensor cycles per stage) need more than 4.
//
// MMA issue: tools/mma_probe.cu measured tcgen05.mma kind::tf32 at N/2 cycles
// per instruction (1190 TFLOP/s at N >= 128) but an issue floor of ~45 cycles
// per instruction even in straight-line code, and 110-150 cycles when each
// instruction recomputes its descriptors and predicate; the issuer therefore
// uses precomputed descriptor bases and literal accumulate flags.
#include <stdlib.h>

#include <algorithm>
#include <type_traits>

#include "gemm_common.cuh"
#include "gemm_engines.cuh"
#include "tc_ptx.cuh"


namespace bf {

int tc2_sacc_max_bn() {
  const char* e = getenv("PURINE_B200_SACC");
  if (e && *e && atoi(e) == 0) return 0;
  const char* m = getenv("PURINE_B200_SACC_MAX_BN");
  return m && *m ? atoi(m) : 128;
}

bool balance_splits_enabled() {
  const char* e = getenv("PURINE_B200_BALANCE_SPLITS");
  return !(e && *e && atoi(e) == 0);
}

bool tc2_wgrad_tma_enabled() {
  if (g_gemm_engine != 0 && g_gemm_engine != 3 && g_gemm_engine != 7) return false;
  static int on = -1;
  if (on < 0) {
    const char* e = getenv("PURINE_B200_WGRAD_TMA");
    on = (e && *e && atoi(e) == 0) ? 0 : 1;
  }
  return on != 0;
}

bool tc2_split_outer() {
  const char* e = getenv("PURINE_B200_SPLIT_OUTER");
  return !(e && *e && atoi(e) == 0);
}

namespace tc2 {

constexpr int BK = 32;
constexpr int STAGES = 8;  // A-ring capacity (barrier arrays); the depth used is w.nst
constexpr int kProducerWarps = 8;
constexpr int kProducers = kProducerWarps * 32;
constexpr int kInvalid = -30000;
constexpr uint32_t kTmemCols = 512;

struct __align__(8) RowInfo {
  int off;
  short h, w;
};

// same separable loader views as engine v1 (gemm_tc.cu)
template <class L>
struct Sep;

template <>
struct Sep<LdFwdX> {
  __device__ static RowInfo row(const LdFwdX& l, int m) {
    const ConvShape& g = l.g;
    int PQ = g.P * g.Q;
    int n = m / PQ, pq = m - n * PQ;
    int p = pq / g.Q, q = pq - p * g.Q;
    int ih = p * g.stride - g.pad, iw = q * g.stride - g.pad;
    return {n * g.C * g.H * g.W + ih * g.W + iw, (short)ih, (short)iw};
  }
  __device__ static RowInfo kin(const LdFwdX& l, int k) {
    const ConvShape& g = l.g;
    int RS = g.R * g.S;
    int c = k / RS, rs = k - c * RS;
    int r = rs / g.S, s = rs - r * g.S;
    return {c * g.H * g.W + r * g.W + s, (short)r, (short)s};
  }
  __device__ static unsigned hb(const LdFwdX& l) { return (unsigned)l.g.H; }
  __device__ static unsigned wb(const LdFwdX& l) { return (unsigned)l.g.W; }
  __device__ static const float* ptr(const LdFwdX& l) { return l.x; }
};

template <>
struct Sep<LdDgradDY> {  // stride 1
  __device__ static RowInfo row(const LdDgradDY& l, int m) {
    const ConvShape& g = l.g;
    int HW = g.H * g.W;
    int n = m / HW, hw = m - n * HW;
    int h = hw / g.W, w = hw - h * g.W;
    int th = h + g.pad, tw = w + g.pad;
    return {n * g.K * g.P * g.Q + th * g.Q + tw, (short)th, (short)tw};
  }
  __device__ static RowInfo kin(const LdDgradDY& l, int k) {
    const ConvShape& g = l.g;
    int RS = g.R * g.S;
    int ko = k / RS, rs = k - ko * RS;
    int r = rs / g.S, s = rs - r * g.S;
    return {ko * g.P * g.Q - r * g.Q - s, (short)-r, (short)-s};
  }
  __device__ static unsigned hb(const LdDgradDY& l) { return (unsigned)l.g.P; }
  __device__ static unsigned wb(const LdDgradDY& l) { return (unsigned)l.g.Q; }
  __device__ static const float* ptr(const LdDgradDY& l) { return l.dy; }
};

template <>
struct Sep<LdWgradX> {  // row = (c,r,s), k = output pixel (n,p,q)
  __device__ static RowInfo row(const LdWgradX& l, int crs) {
    const ConvShape& g = l.g;
    int RS = g.R * g.S;
    int c = crs / RS, rs = crs - c * RS;
    int r = rs / g.S, s = rs - r * g.S;
    return {c * g.H * g.W + r * g.W + s, (short)r, (short)s};
  }
  __device__ static RowInfo kin(const LdWgradX& l, int k) {
    const ConvShape& g = l.g;
    int PQ = g.P * g.Q;
    int n = k / PQ, pq = k - n * PQ;
    int p = pq / g.Q, q = pq - p * g.Q;
    int ih = p * g.stride - g.pad, iw = q * g.stride - g.pad;
    return {n * g.C * g.H * g.W + ih * g.W + iw, (short)ih, (short)iw};
  }
  __device__ static unsigned hb(const LdWgradX& l) { return (unsigned)l.g.H; }
  __device__ static unsigned wb(const LdWgradX& l) { return (unsigned)l.g.W; }
  __device__ static const float* ptr(const LdWgradX& l) { return l.x; }
};

// ---- fast A views: K ordered (r, s, c) with c fastest ----------------------------
// A thread's 16-element chunk is then 16 consecutive input channels at one filter
// tap: one bounds check and a constant address stride per chunk.  Needs the
// channel count divisible by 16 (all GoogLeNet / NIN layers except conv1).

struct ChunkInfo {
  int off;
  short dh, dw;
};

template <class L>
struct Fast {
  __device__ static ChunkInfo chunk(const L&, int) { return {0, 0, 0}; }
  __device__ static int stride(const L&) { return 0; }
  static bool ok(const L&) { return false; }
};

template <>
struct Fast<LdFwdX> {
  __device__ static ChunkInfo chunk(const LdFwdX& l, int kk) {  // kk = first k of the chunk
    const ConvShape& g = l.g;
    int rs = kk / g.C, c0 = kk - rs * g.C;
    int r = rs / g.S, s = rs - r * g.S;
    return {c0 * g.H * g.W + r * g.W + s, (short)r, (short)s};
  }
  __device__ static int stride(const LdFwdX& l) { return l.g.H * l.g.W; }
  static bool ok(const LdFwdX& l) { return l.g.C % 16 == 0; }
};

template <>
struct Fast<LdDgradDY> {
  __device__ static ChunkInfo chunk(const LdDgradDY& l, int kk) {
    const ConvShape& g = l.g;
    int rs = kk / g.K, k0 = kk - rs * g.K;
    int r = rs / g.S, s = rs - r * g.S;
    return {k0 * g.P * g.Q - r * g.Q - s, (short)-r, (short)-s};
  }
  __device__ static int stride(const LdDgradDY& l) { return l.g.P * l.g.Q; }
  static bool ok(const LdDgradDY& l) { return l.g.K % 16 == 0 && l.g.stride == 1; }
};

// weight gradient, fast path: K = pixels ordered (n, p, q) with q padded to Qp
// (Qp = 8 for Q <= 8, else a multiple of 16), so a 16-pixel chunk is one output
// row segment (or two 8-wide rows): per element only compile-time offsets and
// two bounds tests remain.
struct WgradGeom {
  int Pp, Qp;  // padded output rows / cols of the K ordering
};
__host__ inline WgradGeom wgrad_geom(const ConvShape& g) {
  WgradGeom w;
  w.Qp = g.Q <= 8 ? 8 : (g.Q + 15) / 16 * 16;
  const int rpc = 16 / (w.Qp < 16 ? w.Qp : 16);
  w.Pp = (g.P + rpc - 1) / rpc * rpc;
  return w;
}

struct LdWgradDYPad {  // B(n = kout, k' = padded pixel) for the pack kernel
  const float* dy;
  int K, P, Q, Pp, Qp;
  __device__ __forceinline__ float operator()(int ko, int k) const {
    int per = Pp * Qp;
    int n = k / per, rem = k - n * per;
    int p = rem / Qp, q = rem - p * Qp;
    if (p >= P || q >= Q) return 0.f;
    return dy[(((int64_t)n * K + ko) * P + p) * Q + q];
  }
};

// B views with the same (r, s, c) K order for the pack kernel
struct LdFwdWPerm {  // B(n = kout, k' = (rs, c)) = w[kout][c][rs]
  const float* w;
  int C, RS;
  __device__ __forceinline__ float operator()(int n, int k) const {
    int rs = k / C, c = k - rs * C;
    return w[((int64_t)n * C + c) * RS + rs];
  }
};
struct LdDgradWPerm {  // B(n = c, k' = (rs, ko)) = w[ko][c][rs]
  const float* w;
  int C, Kout, RS;
  __device__ __forceinline__ float operator()(int n, int k) const {
    int rs = k / Kout, ko = k - rs * Kout;
    return w[((int64_t)ko * C + n) * RS + rs];
  }
};

using namespace tcu;

// weight-gradient dY pack: a thread owns 4 consecutive padded pixels of one
// row (Qp is a multiple of 8, so they never straddle rows): one decode and one
// float4 load (or 4 scalar loads) per 16-byte chunk instead of per element
__global__ void pack_dy_kernel(LdWgradDYPad lb, int N, int K, int BN, int nkb,
                               uint8_t* __restrict__ out, float* __restrict__ bias_part) {
  const int tile = blockIdx.y, kb = blockIdx.x;
  uint8_t* base = out + ((size_t)tile * nkb + kb) * 2 * BN * 128;
  const int per = lb.Pp * lb.Qp;
  const bool vec = (lb.Q & 3) == 0;
  // the stride (blockDim, a multiple of 8) keeps each thread on one 4-pixel
  // column chunk c: its pixel decode is done once, not per row
  const int c = threadIdx.x & 7;
  const int k0 = kb * BK + c * 4;
  const int n = k0 / per, rem = k0 - n * per;
  const int p = rem / lb.Qp, q = rem - p * lb.Qp;
  for (int i = threadIdx.x; i < BN * 8; i += blockDim.x) {
    const int r = i >> 3;
    const int ko = tile * BN + r;
    float v[4] = {0.f, 0.f, 0.f, 0.f};
    if (ko < N && k0 < K) {
      if (p < lb.P) {
        const float* src = lb.dy + (((int64_t)n * lb.K + ko) * lb.P + p) * lb.Q + q;
        if (vec && q + 3 < lb.Q) {
          const float4 f = __ldg(reinterpret_cast<const float4*>(src));
          v[0] = f.x; v[1] = f.y; v[2] = f.z; v[3] = f.w;
        } else {
#pragma unroll
          for (int j = 0; j < 4; ++j)
            if (q + j < lb.Q) v[j] = __ldg(src + j);
        }
      }
    }
    float4 bg, sm;
    bg.x = to_tf32_rna(v[0]); sm.x = to_tf32_rna(v[0] - bg.x);
    bg.y = to_tf32_rna(v[1]); sm.y = to_tf32_rna(v[1] - bg.y);
    bg.z = to_tf32_rna(v[2]); sm.z = to_tf32_rna(v[2] - bg.z);
    bg.w = to_tf32_rna(v[3]); sm.w = to_tf32_rna(v[3] - bg.w);
    const uint32_t off = sw_off(r, c);
    *reinterpret_cast<float4*>(base + off) = bg;
    *reinterpret_cast<float4*>(base + BN * 128 + off) = sm;
    if (bias_part) {  // fused bias gradient: this k-block's 32-pixel sum per output channel
      float acc = __fadd_rn(__fadd_rn(v[0], v[1]), __fadd_rn(v[2], v[3]));
      acc = __fadd_rn(acc, __shfl_xor_sync(0xffffffffu, acc, 1));
      acc = __fadd_rn(acc, __shfl_xor_sync(0xffffffffu, acc, 2));
      acc = __fadd_rn(acc, __shfl_xor_sync(0xffffffffu, acc, 4));
      if (c == 0 && ko < N) bias_part[(size_t)ko * nkb + kb] = acc;
    }
  }
}

// ---- persistent warp-specialised kernel ---------------------------------------------
//
// warps 0-7   : producers — A gather -> split -> tcgen05.st into the stage's TMEM
//               columns (the next k-block's gathers are issued before the current
//               one is split and stored, so two k-blocks of loads are in flight);
//               thread 0 also streams the stage's packed B tile by TMA
// warp  8     : MMA issuer (one elected thread) + TMEM allocator
// warps 9-16  : epilogue — TMEM accumulator -> registers -> global stores
//               (two warps per TMEM lane quarter, each half of the columns)
//
// Work units (m-tile, n-tile, k-split) are dealt round-robin to a grid of at
// most one CTA per SM; the stage ring (full/empty) runs continuously across
// units and the accumulator is double-buffered when BN <= 128, so the
// epilogue of unit u overlaps the mainloop of unit u+1.

#ifndef TC2_EPI_WARPS
#define TC2_EPI_WARPS 8
#endif
#ifndef TC2_TRUNC_SPLIT
#define TC2_TRUNC_SPLIT 1
#endif
// one tcgen05.commit per k-block: the A and B rings have the same depth and
// the B loader recycles a stage on the A ring's release barrier (each commit
// costs the single issuing thread ~130 cycles, profiles/r01_mma_probe.md)
#ifndef TC2_ONE_COMMIT
#define TC2_ONE_COMMIT 1
#endif
#if TC2_ONE_COMMIT
#define TC2_BRELEASE empty
#else
#define TC2_BRELEASE bempty
#endif
#ifndef TC2_MAX_NST
#define TC2_MAX_NST 7
#endif
constexpr int kEpiWarps = TC2_EPI_WARPS;
constexpr int kMmaWarp = kProducerWarps;
constexpr int kBWarp = kProducerWarps + 1 + kEpiWarps;  // B-tile loader (TMA issue)
constexpr int kAllThreads = (kBWarp + 1) * 32;
constexpr int kBStagesMax = 8;  // B ring depth, independent of the 4-stage TMEM A ring
constexpr int kKtabMax = 4096;  // k-table entries cached in shared memory per CTA

struct Work {
  int M, N, K, BN, nst, nkb, kbps, splits, mtiles, ntiles, units, nacc, full_ktab;
  int nbst;   // B ring stages
  int abase;  // first TMEM column of the A ring
  int accs;   // TMEM column stride between the accumulator buffers
  int sacc;   // 1: separate small-term accumulator in columns [BN, 2BN) of each buffer
  int Pp, Qp;  // weight-gradient fast path: padded pixel grid of the K ordering
  int sstride;  // bytes between ring stages (B tile [+ raw A tile in kTma1x1])
  int cpi;      // kTma1x1 / kWgradTma: 32-pixel k-blocks per image
  // kWgradTma: 0 = dY as [N][K][PQ] (unpadded grid, PQ % 32 == 0); 1 = dY as
  // [N][K][P][Q] with a box of Qp/32-row or 32-column pieces of the padded grid
  int tma4;
  // weight-gradient fast path: x / (Pp*Qp) = (x * per_m) >> per_s, x / Qp likewise
  uint64_t per_m, qp_m;
  int per_s, qp_s;
  // weight gradients: units ordered split-major (m-tile fastest), so the
  // m-tiles sharing a k-range -- and its dY tiles -- run at the same time and
  // the dY pack is read from L2 once per k-range instead of once per m-tile
  int split_outer;
};

// multiply-shift constants for exact unsigned division by d of any x < 2^31
// (m = ceil(2^(31+l) / d), l = ceil(log2 d); m*d - 2^(31+l) < d <= 2^l)
inline void divmagic(uint32_t d, uint64_t& m, int& s) {
  int l = 0;
  while ((1ull << l) < d) ++l;
  s = 31 + l;
  m = ((1ull << s) + d - 1) / d;
}

// TMEM map: nacc accumulator buffers of accs columns, then the A ring.  With
// BN <= 128 the buffers carry a separate small-term accumulator (sacc, see the
// MMA issuer): two 2*BN-column buffers while a >= 4-stage ring remains (BN <=
// 64), else one (BN 96 / 128: measured as fast as two plain buffers).
inline void setup_tmem(Work& w, int nacc_default, int max_nst) {
  w.sacc = (w.BN <= tc2_sacc_max_bn()) ? 1 : 0;
  // two 2*BN buffers only while a >= 4-stage ring remains
  w.nacc = w.sacc ? (4 * w.BN + 256 <= 512 ? 2 : 1) : nacc_default;
  w.accs = w.sacc ? 2 * w.BN : w.BN;  // multiple of 32
  w.abase = (w.nacc * w.accs + 63) / 64 * 64;
  w.nst = std::min<int>(max_nst, (512 - w.abase) / 64);
}

// MODE: 0 generic table gather, 1 channel-chunk fast path (fwd / dgrad),
//       2 / 3 weight-gradient pixel-row fast path with 16- / 8-wide chunks
//       4 TMA-fed 1x1 weight gradient (both operands K-major NCHW tiles, no pack)
//       5 weight gradient with the kWgrad16 gather for A and the raw dY tile
//         streamed by TMA for B (small part split in-kernel, no dY pack):
//         pixel rows exactly 16-aligned and images a whole number of k-blocks
enum { kGeneric = 0, kChannel = 1, kWgrad16 = 2, kWgrad8 = 3, kTma1x1 = 4, kWgradTma = 5 };

// q = x / d, r = x % d, with the (common, warp-uniform) d == 1 case free
__device__ __forceinline__ void divmod_u(int x, int d, int& q, int& r) {
  if (d == 1) {
    q = x;
    r = 0;
  } else {
    q = x / d;
    r = x - q * d;
  }
}
__device__ __forceinline__ void unit_coords(const Work& w, int u, int& mt, int& nt, int& sp) {
  int r;
  if (w.split_outer) {  // u = (sp * ntiles + nt) * mtiles + mt
    divmod_u(u, w.mtiles, r, mt);
    divmod_u(r, w.ntiles, sp, nt);
    return;
  }
  divmod_u(u, w.splits, r, sp);
  divmod_u(r, w.ntiles, mt, nt);
}

__device__ __forceinline__ float ldg_pred(const float* p, int ok) {
  float v;
  asm("{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %2, 0;\n\tmov.b32 %0, 0;\n\t"
      "@q ld.global.nc.f32 %0, [%1];\n\t}"
      : "=f"(v)
      : "l"(p), "r"(ok));
  return v;
}

// Where a gathered element goes: RegSink loads it into a register now;
// AsyncSink issues a 4-byte cp.async (zero-filled when out of bounds) into the
// thread's own column of a shared-memory staging slot, read back by the same
// thread AD k-blocks later (loads in flight without holding registers).
struct RegSink {
  float (&v)[16];
  __device__ __forceinline__ void operator()(int j, const float* p, int ok) const {
    v[j] = ldg_pred(p, ok);
  }
};
struct AsyncSink {
  uint32_t dst;  // smem address of element 0; element j at dst + j * kProducers * 4
  __device__ __forceinline__ void operator()(int j, const float* p, int ok) const {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(dst + j * kProducers * 4),
                 "l"(p), "r"(ok ? 4 : 0)
                 : "memory");
  }
};

template <class SA, bool kTable, class LA, class Sink>
__device__ __forceinline__ void gather16_impl(const LA& la, const Work& w, const RowInfo* ktab,
                                              const RowInfo& ri, int kbase, int kc0,
                                              const float* __restrict__ pa, unsigned hb,
                                              unsigned wb, const Sink& out) {
  if constexpr (kTable) {
    // the 16 table entries (the same for the whole warp: broadcast) come in as
    // 8 x 16-byte shared loads; both bounds tests are evaluated branch-free
    // (a short-circuit && made ptxas predicate the second entry load and
    // reload the bounds from constant memory per element)
    const uint32_t kt = smem_u32(ktab + kbase + kc0);
#pragma unroll
    for (int j2 = 0; j2 < 16; j2 += 2) {
      int off0, hw0, off1, hw1;
      asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];"
                   : "=r"(off0), "=r"(hw0), "=r"(off1), "=r"(hw1)
                   : "r"(kt + j2 * 8));
#pragma unroll
      for (int h2 = 0; h2 < 2; ++h2) {
        const int off = h2 ? off1 : off0, hw = h2 ? hw1 : hw0;
        const int kh = (int)(short)(hw & 0xffff), kw = hw >> 16;
        const int ok = ((unsigned)(ri.h + kh) < hb) & ((unsigned)(ri.w + kw) < wb);
        out(j2 + h2, pa + (ok ? ri.off + off : 0), ok);
      }
    }
    return;
  }
#pragma unroll
  for (int j = 0; j < 16; ++j) {
    const int k = kbase + kc0 + j;
    RowInfo ki;
    if (kTable)
      ki = ktab[k];
    else
      ki = k < w.K ? SA::kin(la, k) : RowInfo{0, (short)kInvalid, (short)kInvalid};
    const int ok = (unsigned)(ri.h + ki.h) < hb && (unsigned)(ri.w + ki.w) < wb;
    out(j, pa + (ok ? ri.off + ki.off : 0), ok);
  }
}

// fast path: the chunk is 16 consecutive channels at one filter tap
template <class LA, class Sink>
__device__ __forceinline__ void gather16_fast(const LA& la, const RowInfo* ktab,
                                              const RowInfo& ri, int kbase, int kc0,
                                              const float* __restrict__ pa, unsigned hb,
                                              unsigned wb, const Sink& out) {
  const ChunkInfo ci = reinterpret_cast<const ChunkInfo*>(ktab)[(kbase + kc0) >> 4];
  const int ok = (unsigned)(ri.h + ci.dh) < hb && (unsigned)(ri.w + ci.dw) < wb;
  const float* p = pa + (ok ? ri.off + ci.off : 0);
  const int stride = Fast<LA>::stride(la);
#pragma unroll
  for (int j = 0; j < 16; ++j) out(j, p + j * stride, ok);
}

template <int CCW, class LA, class Sink>
__device__ __forceinline__ void gather16_wgrad(const LA& la, const Work& w, const RowInfo& ri,
                                               int kk, const float* __restrict__ pa,
                                               const Sink& out) {
  const ConvShape& g = la.g;
  // (n, p0, q0) of pixel kk by multiply-shift division (Work::per_m / qp_m,
  // exact for kk < 2^31): a runtime integer divide was ~20 instructions, twice
  // per 16 elements on the issue-bound producers (weight gradients 4.64 ->
  // 4.40 ms).  A per-row [jlo, jhi) column range test with pointer selects
  // instead of the per-element bounds tests measured 10% slower.
  const int n = (int)(((uint64_t)(uint32_t)kk * w.per_m) >> w.per_s);
  const int rem = kk - n * w.Pp * w.Qp;
  const int p0 = (int)(((uint64_t)(uint32_t)rem * w.qp_m) >> w.qp_s);
  const int q0 = rem - p0 * w.Qp;
  const int st = g.stride;
  const int ihb = p0 * st - g.pad + ri.h, iwb = q0 * st - g.pad + ri.w;
  const int64_t off0 =
      (int64_t)n * g.C * g.H * g.W + ri.off + (p0 * st - g.pad) * g.W + (q0 * st - g.pad);
  const bool live = kk < w.K;
#pragma unroll
  for (int j = 0; j < 16; ++j) {
    const int jr = j / CCW, jc = j % CCW;
    const int ih = ihb + jr * st, iw = iwb + jc * st;
    const int ok = live && (p0 + jr < g.P) && (q0 + jc < g.Q) && (unsigned)ih < (unsigned)g.H &&
                   (unsigned)iw < (unsigned)g.W;
    out(j, pa + (ok ? off0 + (int64_t)jr * st * g.W + jc * st : 0), ok);
  }
}

// A operand split for 3xTF32: big = x as is (the MMA reads it as trunc(x)),
// small = tf32_small(x) (tc_ptx.cuh: x - trunc(x), rounded to nearest by the
// MMA's own truncation).  TC2_TRUNC_SPLIT=0 selects the explicit
// round-to-nearest split (2 more integer ops per element).
__device__ __forceinline__ void split_tf32(float x, float& big, float& small) {
#if TC2_TRUNC_SPLIT
  big = x;
  small = tf32_small(x);
#else
  big = to_tf32_rna(x);
  small = to_tf32_rna(x - big);
#endif
}

// the table/no-table choice is hoisted out of the unrolled loop so the
// division-heavy fallback is never if-converted into the common path
template <class SA, int MODE, class LA, class Sink>
__device__ __forceinline__ void gather16_to(const LA& la, const Work& w, const RowInfo* ktab,
                                            const RowInfo& ri, int kbase, int kc0,
                                            const float* __restrict__ pa, unsigned hb,
                                            unsigned wb, const Sink& out) {
  if (MODE == kWgrad16 || MODE == kWgradTma)
    gather16_wgrad<16>(la, w, ri, kbase + kc0, pa, out);
  else if (MODE == kWgrad8)
    gather16_wgrad<8>(la, w, ri, kbase + kc0, pa, out);
  else if (MODE == kChannel)
    gather16_fast(la, ktab, ri, kbase, kc0, pa, hb, wb, out);
  else if (w.full_ktab)
    gather16_impl<SA, true>(la, w, ktab, ri, kbase, kc0, pa, hb, wb, out);
  else
    gather16_impl<SA, false>(la, w, ktab, ri, kbase, kc0, pa, hb, wb, out);
}
template <class SA, int MODE, class LA>
__device__ __forceinline__ void gather16(const LA& la, const Work& w, const RowInfo* ktab,
                                         const RowInfo& ri, int kbase, int kc0,
                                         const float* __restrict__ pa, unsigned hb, unsigned wb,
                                         float (&v)[16]) {
  gather16_to<SA, MODE>(la, w, ktab, ri, kbase, kc0, pa, hb, wb, RegSink{v});
}

// AD > 0: the producers' gathers run AD k-blocks ahead through cp.async into a
// shared-memory staging ring (AD x 16 KB) instead of one k-block ahead in
// registers (which is all the 17-warp register budget allows)
template <class LA, class Epi, int MODE, int AD = 0>
__global__ void __launch_bounds__(kAllThreads, 1)
    tc2_kernel(LA la, Work w, const uint8_t* __restrict__ bpack, Epi epi, EpiPartial part,
               const __grid_constant__ CUtensorMap amap, const __grid_constant__ CUtensorMap bmap,
               float* __restrict__ bias_part) {
  using SA = Sep<LA>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  const int BN = w.BN;
  const int stage_bytes = 2 * BN * 128;
  uint8_t* tiles = base;
  const int ktab_n = w.full_ktab ? w.nkb * BK : STAGES * BK;
  const int sstride = w.sstride;
  float* staging = reinterpret_cast<float*>(base + w.nbst * sstride);  // AD x [16][kProducers]
  RowInfo* ktab = reinterpret_cast<RowInfo*>(base + w.nbst * sstride + AD * 16 * kProducers * 4);
  uint64_t* full = reinterpret_cast<uint64_t*>(ktab + ktab_n);
  uint64_t* empty = full + STAGES;
  uint64_t* bfull = empty + STAGES;
  uint64_t* bempty = bfull + kBStagesMax;
  uint64_t* acc_full = bempty + kBStagesMax;
  uint64_t* acc_empty = acc_full + 2;
  uint64_t* bsplit = acc_empty + 2;  // kWgradTma: the epilogue warps split the raw B tile
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bsplit + kBStagesMax);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (warp == kMmaWarp) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)),
                 "r"(kTmemCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], kProducers);
      mbar_init(&empty[s], 1);
    }
    for (int s = 0; s < kBStagesMax; ++s) {
      mbar_init(&bfull[s], 1);
      mbar_init(&bempty[s], 1);
      mbar_init(&bsplit[s], kEpiWarps * 32);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&acc_full[b], 1);
      mbar_init(&acc_empty[b], kEpiWarps * 32);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (MODE == kChannel) {  // per 16-channel chunk: offset and filter tap, once per CTA
    ChunkInfo* ct = reinterpret_cast<ChunkInfo*>(ktab);
    for (int c = threadIdx.x; c < ktab_n / 16; c += kAllThreads)
      ct[c] = c * 16 < w.K ? Fast<LA>::chunk(la, c * 16)
                           : ChunkInfo{0, (short)kInvalid, (short)kInvalid};
  } else if (MODE == kGeneric && w.full_ktab) {  // k -> gather offsets, whole K, once per CTA
    for (int k = threadIdx.x; k < ktab_n; k += kAllThreads)
      ktab[k] = k < w.K ? SA::kin(la, k) : RowInfo{0, (short)kInvalid, (short)kInvalid};
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp < kProducerWarps) {
    // ======================= producers =======================
    const int t = threadIdx.x;
    const int q = warp & 3;
    const int kc0 = (warp >> 2) * 16;
    const float* __restrict__ pa = SA::ptr(la);
    const unsigned hb = SA::hb(la), wb = SA::wb(la);
    const uint32_t lane_addr = tmem + ((uint32_t)(q * 32) << 16);
    auto row_of = [&](int u) {
      int mt, nt, sp;
      unit_coords(w, u, mt, nt, sp);
      const int m = mt * BM + q * 32 + lane;
      return m < w.M ? SA::row(la, m) : RowInfo{0, (short)kInvalid, (short)kInvalid};
    };
    int u = blockIdx.x, i = 0, it = 0;
    if (MODE == kTma1x1) {
      // A (x rows) and B (dy rows) arrive as raw fp32 tiles by TMA.  Each
      // thread splits its TMEM lane's 16 A values (4 swizzled 16-byte chunks
      // of row m) into big/small for TMEM, writes the small part of BN/32 of
      // the B tile's 16-byte chunks next to the raw tile (raw = big: the tensor
      // core drops the low 13 bits itself) and, for m-tile 0, sums those dy
      // chunks into per-row bias partials.
      const int m_row = q * 32 + lane;
      const int nb = BN / 32;  // 16-byte B chunks per thread per stage
      int bs = 0, stage = 0;
      uint32_t bph = 0, ph = 0;
      for (; u < w.units; u += gridDim.x) {
        int mt, nt, sp;
        unit_coords(w, u, mt, nt, sp);
        const int kb0 = sp * w.kbps;
        const int nk = min(w.kbps, w.nkb - kb0);
        const bool do_bias = bias_part != nullptr && mt == 0;
        float bsum[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) bsum[j] = 0.f;
        for (int i2 = 0; i2 < nk; ++i2) {
          mbar_wait(&bfull[bs], bph);
          uint8_t* sb = tiles + bs * sstride;
          const uint8_t* araw = sb + 2 * BN * 128;
          float big[16], small[16];
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            const int chunk = (kc0 >> 2) + c;
            const float4 v = *reinterpret_cast<const float4*>(araw + m_row * 128 +
                                                              ((chunk ^ (m_row & 7)) << 4));
            split_tf32(v.x, big[4 * c + 0], small[4 * c + 0]);
            split_tf32(v.y, big[4 * c + 1], small[4 * c + 1]);
            split_tf32(v.z, big[4 * c + 2], small[4 * c + 2]);
            split_tf32(v.w, big[4 * c + 3], small[4 * c + 3]);
          }
          const float4* braw = reinterpret_cast<const float4*>(sb);
          float4* bsm = reinterpret_cast<float4*>(sb + BN * 128);
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            if (j < nb) {
              const int f = t + kProducers * j;
              const float4 v = braw[f];
              const float4 r = tf32_small4(v);
              bsm[f] = r;
              if (do_bias)
                bsum[j] = __fadd_rn(bsum[j], __fadd_rn(__fadd_rn(v.x, v.y), __fadd_rn(v.z, v.w)));
            }
          }
          // generic-proxy smem writes -> visible to the tensor core (async proxy)
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          mbar_wait(&empty[stage], ph ^ 1);
          const uint32_t acol = w.abase + stage * 64 + kc0;
          tmem_st16(lane_addr + acol, big);
          tmem_st16(lane_addr + acol + 32, small);
          asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
          tc_fence_before();
          mbar_arrive(&full[stage]);
          if (++bs == w.nbst) {
            bs = 0;
            bph ^= 1;
          }
          if (++stage == w.nst) {
            stage = 0;
            ph ^= 1;
          }
        }
        if (do_bias) {
          // chunk f of the tile is row f / 8: the 8 lanes t^1, t^2, t^4 share a row
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            if (j < nb) {
              float a = bsum[j];
              a = __fadd_rn(a, __shfl_xor_sync(0xffffffffu, a, 1));
              a = __fadd_rn(a, __shfl_xor_sync(0xffffffffu, a, 2));
              a = __fadd_rn(a, __shfl_xor_sync(0xffffffffu, a, 4));
              const int row = nt * BN + (t >> 3) + 32 * j;
              if ((t & 7) == 0 && row < w.N) bias_part[(size_t)row * w.splits + sp] = a;
            }
          }
        }
      }
    } else if (MODE == kGeneric && !w.full_ktab) {
      // K too long for a cached table (weight gradients: K = N*P*Q pixels):
      // the k-block's 32 gather offsets are computed per stage into a ring slot
      int gstage = 0;
      uint32_t gphase = 0;
      for (; u < w.units; u += gridDim.x) {
        int mt, nt, sp;
        unit_coords(w, u, mt, nt, sp);
        const RowInfo ri = row_of(u);
        const int kb0 = sp * w.kbps;
        const int nk = min(w.kbps, w.nkb - kb0);
        for (int i2 = 0; i2 < nk; ++i2, ++it) {
          const int stage = gstage;
          const uint32_t phase = gphase;
          if (++gstage == w.nst) {
            gstage = 0;
            gphase ^= 1;
          }
          const int kbase = (kb0 + i2) * BK;
          RowInfo* slot = ktab + stage * BK;
          if (t < BK) {
            const int k = kbase + t;
            slot[t] = k < w.K ? SA::kin(la, k) : RowInfo{0, (short)kInvalid, (short)kInvalid};
          }
          named_sync(1, kProducers);
          float v[16];
          gather16_impl<SA, true>(la, w, slot - kbase, ri, kbase, kc0, pa, hb, wb, RegSink{v});
          float big[16], small[16];
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            split_tf32(v[j], big[j], small[j]);
          }
          mbar_wait(&empty[stage], phase ^ 1);
          const uint32_t acol = w.abase + stage * 64 + kc0;
          tmem_st16(lane_addr + acol, big);
          tmem_st16(lane_addr + acol + 32, small);
          asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
          tc_fence_before();
          mbar_arrive(&full[stage]);
        }
      }
    } else if (AD > 0 && u < w.units) {
      // issue cursor (iu, ii) runs AD k-blocks ahead of the consume cursor (u, i)
      int iu = u, ii = 0, ikb0, ink;
      RowInfo iri = row_of(iu);
      {
        int mt2, nt2, sp2;
        unit_coords(w, iu, mt2, nt2, sp2);
        ikb0 = sp2 * w.kbps;
        ink = min(w.kbps, w.nkb - ikb0);
      }
      const uint32_t stg = smem_u32(staging) + t * 4;
      auto issue = [&](int slot) {
        if (iu < w.units) {
          gather16_to<SA, MODE>(la, w, ktab, iri, (ikb0 + ii) * BK, kc0, pa, hb, wb,
                                AsyncSink{stg + (uint32_t)(slot * 16 * kProducers * 4)});
          if (++ii >= ink) {
            iu += gridDim.x;
            ii = 0;
            if (iu < w.units) {
              int mt2, nt2, sp2;
              unit_coords(w, iu, mt2, nt2, sp2);
              iri = row_of(iu);
              ikb0 = sp2 * w.kbps;
              ink = min(w.kbps, w.nkb - ikb0);
            }
          }
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
      };
#pragma unroll
      for (int d = 0; d < (AD > 0 ? AD : 1); ++d) issue(d);
      int pstage = 0, slot = 0;
      uint32_t pphase = 0;
      int nk, cmt, cnt_, csp;
      unit_coords(w, u, cmt, cnt_, csp);
      nk = min(w.kbps, w.nkb - csp * w.kbps);
      while (true) {
        asm volatile("cp.async.wait_group %0;" ::"n"(AD > 0 ? AD - 1 : 0) : "memory");
        float big[16], small[16];
        {
          const float* sv = staging + slot * 16 * kProducers + t;
#pragma unroll
          for (int j = 0; j < 16; ++j) split_tf32(sv[j * kProducers], big[j], small[j]);
        }
        issue(slot);  // refill the slot just read (its values are in registers)
        if (++slot == AD) slot = 0;
        const int stage = pstage;
        const uint32_t phase = pphase;
        if (++pstage == w.nst) {
          pstage = 0;
          pphase ^= 1;
        }
        mbar_wait(&empty[stage], phase ^ 1);
        const uint32_t acol = w.abase + stage * 64 + kc0;
        tmem_st16(lane_addr + acol, big);
        tmem_st16(lane_addr + acol + 32, small);
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        tc_fence_before();
        mbar_arrive(&full[stage]);
        if (++i >= nk) {
          u += gridDim.x;
          i = 0;
          if (u >= w.units) break;
          unit_coords(w, u, cmt, cnt_, csp);
          nk = min(w.kbps, w.nkb - csp * w.kbps);
        }
      }
      asm volatile("cp.async.wait_all;" ::: "memory");
    } else if (MODE == kChannel && u < w.units) {
      // channel-chunk gathers (fwd / dgrad): two k-blocks of register
      // prefetch, three buffers used round-robin (the body is instantiated
      // three times with rotated roles: no moves).  Measured: conv2/3x3 data
      // gradient 0.64 -> 0.59 ms; the table-driven generic gather (conv1's
      // forward) is slower with the extra registers, so it keeps one k-block
      int pstage = 0;
      uint32_t pphase = 0;
      int left = 0;  // k-blocks this CTA publishes
      for (int uu = u; uu < w.units; uu += gridDim.x) {
        int mt2, nt2, sp2;
        unit_coords(w, uu, mt2, nt2, sp2);
        left += min(w.kbps, w.nkb - sp2 * w.kbps);
      }
      RowInfo ri = row_of(u);
      int kb0, nk;
      {
        int mt2, nt2, sp2;
        unit_coords(w, u, mt2, nt2, sp2);
        kb0 = sp2 * w.kbps;
        nk = min(w.kbps, w.nkb - kb0);
      }
      auto issue = [&](float (&dst)[16]) {  // gather the issue cursor's k-block, advance it
        if (u >= w.units) return;
        gather16<SA, MODE>(la, w, ktab, ri, (kb0 + i) * BK, kc0, pa, hb, wb, dst);
        if (++i >= nk) {
          u += gridDim.x;
          i = 0;
          if (u < w.units) {
            int mt2, nt2, sp2;
            unit_coords(w, u, mt2, nt2, sp2);
            ri = row_of(u);
            kb0 = sp2 * w.kbps;
            nk = min(w.kbps, w.nkb - kb0);
          }
        }
      };
      float va[16], vb[16], vc[16];
      issue(va);
      issue(vb);
      auto step = [&](float (&cur)[16], float (&pre)[16]) -> bool {
        issue(pre);
        float big[16], small[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) split_tf32(cur[j], big[j], small[j]);
        const int stage = pstage;
        const uint32_t phase = pphase;
        if (++pstage == w.nst) {
          pstage = 0;
          pphase ^= 1;
        }
        mbar_wait(&empty[stage], phase ^ 1);
        const uint32_t acol = w.abase + stage * 64 + kc0;
        tmem_st16(lane_addr + acol, big);
        tmem_st16(lane_addr + acol + 32, small);
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        tc_fence_before();
        mbar_arrive(&full[stage]);
        return --left > 0;
      };
      while (step(va, vc) && step(vb, va) && step(vc, vb)) {
      }
    } else if (u < w.units) {
      // one k-block of register prefetch in two fixed buffers used ping-pong
      // (the loop body is instantiated twice with the roles swapped): a
      // rotation copy v = v2 would stall on the prefetch loads at the end of
      // every k-block (ncu: 9.5% of the conv2 data gradient's samples on that
      // move), i.e. no overlap across the publish step
      int pstage = 0;
      uint32_t pphase = 0;
      RowInfo ri = row_of(u);
      int kb0, nk;
      {
        int mt2, nt2, sp2;
        unit_coords(w, u, mt2, nt2, sp2);
        kb0 = sp2 * w.kbps;
        nk = min(w.kbps, w.nkb - kb0);
      }
      float va[16], vb[16];
      gather16<SA, MODE>(la, w, ktab, ri, kb0 * BK, kc0, pa, hb, wb, va);
      // publishes `cur` (the current k-block), prefetching the next into `nxt`;
      // false once the last k-block is published
      auto step = [&](float (&cur)[16], float (&nxt)[16]) -> bool {
        if (++i >= nk) {
          u += gridDim.x;
          i = 0;
          if (u < w.units) {
            int mt2, nt2, sp2;
            unit_coords(w, u, mt2, nt2, sp2);
            ri = row_of(u);
            kb0 = sp2 * w.kbps;
            nk = min(w.kbps, w.nkb - kb0);
          }
        }
        const bool more = u < w.units;
        if (more) gather16<SA, MODE>(la, w, ktab, ri, (kb0 + i) * BK, kc0, pa, hb, wb, nxt);
        float big[16], small[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) split_tf32(cur[j], big[j], small[j]);
        const int stage = pstage;
        const uint32_t phase = pphase;
        if (++pstage == w.nst) {
          pstage = 0;
          pphase ^= 1;
        }
        mbar_wait(&empty[stage], phase ^ 1);
        const uint32_t acol = w.abase + stage * 64 + kc0;
        tmem_st16(lane_addr + acol, big);
        tmem_st16(lane_addr + acol + 32, small);
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        tc_fence_before();
        mbar_arrive(&full[stage]);
        return more;
      };
      while (step(va, vb) && step(vb, va)) {
      }
    }
  } else if (warp == kMmaWarp) {
    // ======================= MMA issuer =======================
    // the whole warp walks the schedule and waits (convergent, so the
    // operands reach tcgen05.mma as warp-uniform values); one elected lane
    // issues the MMAs and their commits.  (A lane-0-only loop with any data-
    // dependent branch made ptxas emit an illegal uniform-register sequence.)
    {
      const uint32_t idesc = tf32_idesc(BN);
      const uint32_t idesc2 = tf32_idesc(w.sacc ? 2 * BN : BN);
      const uint64_t dtiles = sw128_desc(smem_u32(tiles));  // B stage 0, big image, k-step 0
      const uint64_t dsmall = (uint64_t)((BN * 128) >> 4);   // big -> small image
      // ring positions advance incrementally: a runtime modulo / divide per
      // k-block cost the single issuing warp ~80 instructions
      int stage = 0, bst = 0, local = 0;
      uint32_t phase = 0, bphase = 0;
      for (int u = blockIdx.x; u < w.units; u += gridDim.x, ++local) {
        int mt, nt, sp;
        unit_coords(w, u, mt, nt, sp);
        const int nk = min(w.kbps, w.nkb - sp * w.kbps);
        const int b = local % w.nacc;
        const uint32_t use = local / w.nacc;
        mbar_wait(&acc_empty[b], (use & 1) ^ 1);
        tc_fence_after();
        const uint32_t dacc = tmem + (uint32_t)(b * w.accs);
        for (int i = 0; i < nk; ++i) {
          // kWgradTma: the raw tile landed AND its small half is written
          mbar_wait(MODE == kWgradTma ? &bsplit[bst] : &bfull[bst], bphase);
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          // descriptor start-address field = smem byte address >> 4 (bits 0-13)
          const uint64_t db = dtiles + (uint64_t)((bst * sstride) >> 4);
          const uint64_t ds = db + dsmall;
          const uint32_t ab = tmem + w.abase + stage * 64;
          if (elect_one()) {
            if (w.sacc) {
              // the B stage is [B big rows | B small rows]: one N = 2*BN MMA puts
              // A_big*B_big in columns [0, BN) and A_big*B_small in [BN, 2BN),
              // where A_small*B_big accumulates too -- two instructions per
              // k-step, and one round-toward-zero accumulation of the big
              // accumulator instead of three (tc4 measured 2.3x less error)
              const uint32_t dsm = dacc + (uint32_t)BN;
              if (i == 0)
                mma_ts_flag<0>(dacc, ab, db, idesc2);
              else
                mma_ts_flag<1>(dacc, ab, db, idesc2);
              mma_ts_flag<1>(dsm, ab + 32, db, idesc);
#pragma unroll
              for (int ks = 1; ks < BK / 8; ++ks) {
                const uint64_t k2 = (uint64_t)((ks * 32) >> 4);
                mma_ts_flag<1>(dacc, ab + ks * 8, db + k2, idesc2);
                mma_ts_flag<1>(dsm, ab + 32 + ks * 8, db + k2, idesc);
              }
            } else {
            // 3xTF32 per k-step of 8: small*big + big*small + big*big
            if (i == 0)
              mma_ts_flag<0>(dacc, ab + 32, db, idesc);
            else
              mma_ts_flag<1>(dacc, ab + 32, db, idesc);
            mma_ts_flag<1>(dacc, ab, ds, idesc);
            mma_ts_flag<1>(dacc, ab, db, idesc);
#pragma unroll
            for (int ks = 1; ks < BK / 8; ++ks) {
              const uint64_t k2 = (uint64_t)((ks * 32) >> 4);
              mma_ts_flag<1>(dacc, ab + 32 + ks * 8, db + k2, idesc);
              mma_ts_flag<1>(dacc, ab + ks * 8, ds + k2, idesc);
              mma_ts_flag<1>(dacc, ab + ks * 8, db + k2, idesc);
            }
            }
            tc_commit(&empty[stage]);
#if !TC2_ONE_COMMIT
            tc_commit(&bempty[bst]);
#endif
          }
          __syncwarp();
          if (++stage == w.nst) {
            stage = 0;
            phase ^= 1;
          }
          if (++bst == w.nbst) {
            bst = 0;
            bphase ^= 1;
          }
        }
        if (elect_one()) tc_commit(&acc_full[b]);
        __syncwarp();
      }
    }
  } else if (warp == kBWarp) {
    // ======================= B loader =======================
    // streams the pre-packed B tiles of every (unit, k-block) into the B ring
    // as far ahead as the ring allows: the TMA latency leaves the per-stage
    // critical path of the producers
    if (MODE == kWgradTma && lane == 0) {
      // raw dy tile (BN rows x 32 pixels) of each k-block; k-blocks never
      // straddle images (launch_wgrad_tma checks PQ % 32 == 0)
      int bst = 0;
      uint32_t bphase = 0;
      for (int u = blockIdx.x; u < w.units; u += gridDim.x) {
        int mt, nt, sp;
        unit_coords(w, u, mt, nt, sp);
        const int kb0 = sp * w.kbps;
        const int nk = min(w.kbps, w.nkb - kb0);
        for (int i = 0; i < nk; ++i) {
          mbar_wait(&TC2_BRELEASE[bst], bphase ^ 1);
          mbar_arrive_expect_tx(&bfull[bst], (uint32_t)(BN * 128));
          const int kb = kb0 + i, img = kb / w.cpi, j = kb - img * w.cpi;
          if (w.tma4) {
            // padded grid Pp x Qp: a k-block is 32 / Qp whole rows (Qp <= 32)
            // or a 32-column piece of one row; pixels past P / Q read as zero
            int p0, q0;
            if (w.Qp <= BK) {
              p0 = j * (BK / w.Qp);
              q0 = 0;
            } else {
              const int per_row = w.Qp / BK;
              p0 = j / per_row;
              q0 = (j - p0 * per_row) * BK;
            }
            tma_load_4d(smem_u32(tiles + bst * sstride), &bmap, q0, p0, nt * BN, img,
                        &bfull[bst]);
          } else {
            tma_load_3d(smem_u32(tiles + bst * sstride), &bmap, j * BK, nt * BN, img,
                        &bfull[bst]);
          }
          if (++bst == w.nbst) {
            bst = 0;
            bphase ^= 1;
          }
        }
      }
    } else if (MODE == kTma1x1 && lane == 0) {
      // raw dy tile (BN rows) and x tile (BM rows) of one 32-pixel k-block
      int bst = 0;
      uint32_t bphase = 0;
      for (int u = blockIdx.x; u < w.units; u += gridDim.x) {
        int mt, nt, sp;
        unit_coords(w, u, mt, nt, sp);
        const int kb0 = sp * w.kbps;
        const int nk = min(w.kbps, w.nkb - kb0);
        for (int i = 0; i < nk; ++i) {
          mbar_wait(&TC2_BRELEASE[bst], bphase ^ 1);
          mbar_arrive_expect_tx(&bfull[bst], (uint32_t)(BN * 128 + BM * 128));
          const int kb = kb0 + i, img = kb / w.cpi, pix = (kb - img * w.cpi) * BK;
          uint8_t* sb = tiles + bst * sstride;
          tma_load_3d(smem_u32(sb), &bmap, pix, nt * BN, img, &bfull[bst]);
          tma_load_3d(smem_u32(sb + 2 * BN * 128), &amap, pix, mt * BM, img, &bfull[bst]);
          if (++bst == w.nbst) {
            bst = 0;
            bphase ^= 1;
          }
        }
      }
    } else if (lane == 0) {
      int bst = 0;
      uint32_t bphase = 0;
      for (int u = blockIdx.x; u < w.units; u += gridDim.x) {
        int mt, nt, sp;
        unit_coords(w, u, mt, nt, sp);
        const int kb0 = sp * w.kbps;
        const int nk = min(w.kbps, w.nkb - kb0);
        for (int i = 0; i < nk; ++i) {
          mbar_wait(&TC2_BRELEASE[bst], bphase ^ 1);
          mbar_arrive_expect_tx(&bfull[bst], (uint32_t)stage_bytes);
          bulk_g2s(smem_u32(tiles + bst * sstride),
                   bpack + ((size_t)nt * w.nkb + kb0 + i) * stage_bytes, (uint32_t)stage_bytes,
                   &bfull[bst]);
          if (++bst == w.nbst) {
            bst = 0;
            bphase ^= 1;
          }
        }
      }
    }
    __syncwarp();
  } else {
    // ======================= epilogue =======================
    const int ew = warp - kMmaWarp - 1;  // 0..kEpiWarps-1
    const int q = warp & 3;
    const int half = kEpiWarps == 8 ? (ew >> 2) : 0;
    auto drain = [&](int u, int local) {
      int mt, nt, sp;
      unit_coords(w, u, mt, nt, sp);
      const int b = local % w.nacc;
      const uint32_t use = local / w.nacc;
      mbar_wait(&acc_full[b], use & 1);
      tc_fence_after();
      const int m = mt * BM + q * 32 + lane;
      const int n0 = nt * BN;
      const int cols = kEpiWarps == 8 ? BN / 2 : BN;
      const uint32_t taddr = tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(b * w.accs);
      const bool live = m < w.M;
      const RowPtr rp = live ? (w.splits > 1 ? part.row(sp, m) : epi.row(m)) : RowPtr{nullptr, 0.f};
#pragma unroll 1
      for (int c0 = half * cols; c0 < half * cols + cols; c0 += 16) {
        uint32_t v[16];
        tmem_ld16(taddr + (uint32_t)c0, v);
        if (w.sacc) {  // big + small halves, fp32 round-to-nearest
          uint32_t sv[16];
          tmem_ld16(taddr + (uint32_t)(BN + c0), sv);
#pragma unroll
          for (int j = 0; j < 16; ++j)
            v[j] = __float_as_uint(__fadd_rn(__uint_as_float(v[j]), __uint_as_float(sv[j])));
        }
        if (live) {
          const int nlim = w.N - (n0 + c0);
          if (w.splits > 1) {
            part.store16(rp, n0 + c0, v, nlim);
          } else {
            epi.store16(rp, n0 + c0, v, nlim);
          }
        }
      }
      tc_fence_before();
      mbar_arrive(&acc_empty[b]);
    };
    if constexpr (MODE == kWgradTma) {
      // The epilogue warps, idle between accumulator drains in a weight
      // gradient, also turn each raw dY tile (TMA) into the B stage: its
      // small part next to it (the raw tile is the big part: the tensor core
      // drops the low 13 bits itself) and, for m-tile 0, its per-row sums into
      // the bias partials -- no dY pack pass, and none of it on the issue-bound
      // im2col producers.  Drains interleave with the splits: before blocking
      // on a tile whose TMA waits for the MMA to free its stage, a unit whose
      // k-blocks are all split is drained as soon as its accumulator is ready
      // (the MMA may be waiting for that buffer).
      static_assert(MODE != kWgradTma || kEpiWarps == 8,
                    "the B split maps 256 epilogue threads onto the tile");
      const int te = threadIdx.x - (kMmaWarp + 1) * 32;  // 0..255
      const int nb = BN / 32;
      int su = blockIdx.x, si = 0, s_nk = 0, s_mt = 0, s_nt = 0, s_sp = 0;
      auto load_unit = [&]() {
        if (su < w.units) {
          unit_coords(w, su, s_mt, s_nt, s_sp);
          s_nk = min(w.kbps, w.nkb - s_sp * w.kbps);
        }
      };
      load_unit();
      int bst = 0, du = blockIdx.x, dlocal = 0, split_done = 0;
      uint32_t bphase = 0;
      float bsum[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) bsum[j] = 0.f;
      while (su < w.units || du < w.units) {
        if (du < w.units && dlocal < split_done) {
          bool ready = su >= w.units;
          if (!ready) {
            uint32_t ok = 0;
            const int b = dlocal % w.nacc;
            asm volatile(
                "{\n\t.reg .pred P1;\n\tmbarrier.test_wait.parity.shared::cta.b64 P1, [%1], %2;"
                "\n\tselp.u32 %0, 1, 0, P1;\n\t}"
                : "=r"(ok)
                : "r"(smem_u32(&acc_full[b])), "r"((uint32_t)((dlocal / w.nacc) & 1))
                : "memory");
            ready = __shfl_sync(0xffffffffu, ok, 0) != 0;
          }
          if (ready) {
            drain(du, dlocal);
            du += gridDim.x;
            ++dlocal;
            continue;
          }
        }
        if (su >= w.units) continue;
        {
          uint32_t ok = 0;
          asm volatile(
              "{\n\t.reg .pred P1;\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;"
              "\n\tselp.u32 %0, 1, 0, P1;\n\t}"
              : "=r"(ok)
              : "r"(smem_u32(&bfull[bst])), "r"(bphase)
              : "memory");
          if (__shfl_sync(0xffffffffu, ok, 0) == 0) continue;  // timed out: poll the drain
        }
        mbar_wait(&bfull[bst], bphase);  // complete: acquire for every lane
        {
          uint8_t* sb = tiles + bst * sstride;
          const float4* braw = reinterpret_cast<const float4*>(sb);
          float4* bsm = reinterpret_cast<float4*>(sb + BN * 128);
          const bool do_bias = bias_part != nullptr && s_mt == 0;
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            if (j < nb) {
              const int f = te + kEpiWarps * 32 * j;
              const float4 v = braw[f];
              bsm[f] = tf32_small4(v);
              if (do_bias)
                bsum[j] = __fadd_rn(bsum[j], __fadd_rn(__fadd_rn(v.x, v.y), __fadd_rn(v.z, v.w)));
            }
          }
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          mbar_arrive(&bsplit[bst]);
        }
        if (++bst == w.nbst) {
          bst = 0;
          bphase ^= 1;
        }
        if (++si >= s_nk) {
          if (bias_part != nullptr && s_mt == 0) {
            // 16-byte chunk f of the tile is row f / 8: lanes te^1, te^2, te^4 share a row
#pragma unroll
            for (int j = 0; j < 8; ++j) {
              if (j < nb) {
                float a = bsum[j];
                a = __fadd_rn(a, __shfl_xor_sync(0xffffffffu, a, 1));
                a = __fadd_rn(a, __shfl_xor_sync(0xffffffffu, a, 2));
                a = __fadd_rn(a, __shfl_xor_sync(0xffffffffu, a, 4));
                const int row = s_nt * BN + (te >> 3) + 32 * j;
                if ((te & 7) == 0 && row < w.N) bias_part[(size_t)row * w.splits + s_sp] = a;
                bsum[j] = 0.f;
              }
            }
          }
          ++split_done;
          su += gridDim.x;
          si = 0;
          load_unit();
        }
      }
    } else {
      int local = 0;
      for (int u = blockIdx.x; u < w.units; u += gridDim.x, ++local) drain(u, local);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == kMmaWarp) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                 "r"(kTmemCols));
  }
}

inline int pick_bn(int N, int& ntiles) {
  ntiles = (N + 255) / 256;
  int per = (N + ntiles - 1) / ntiles;
  return (per + 31) / 32 * 32;
}

template <class LA, class LB, class LBP, class Epi>
int launch(const LA& la, const LB& lb, const LBP& lbp, int M, int N, int K, const Epi& epi,
           float* ws, int64_t ws_bytes, cudaStream_t st, const char* what, int mode = -1,
           int Pp = 0, int Qp = 0, float* bias_out = nullptr) {
  if (mode < 0) mode = Fast<LA>::ok(la) ? kChannel : kGeneric;
  const bool fast = mode != kGeneric;
  Work w{};
  w.M = M;
  w.N = N;
  w.K = K;
  w.Pp = Pp;
  w.Qp = Qp;
  if (Pp > 0 && Qp > 0) {
    divmagic((uint32_t)(Pp * Qp), w.per_m, w.per_s);
    divmagic((uint32_t)Qp, w.qp_m, w.qp_s);
  }
  w.BN = pick_bn(N, w.ntiles);
  w.nkb = (K + BK - 1) / BK;
  w.mtiles = (M + BM - 1) / BM;
#ifndef TC2_NACC1_MIN_KB
#define TC2_NACC1_MIN_KB 1000000000
#endif
  // one accumulator (a deeper TMEM A ring) for long k loops, where the ring
  // depth bounds throughput and the epilogue is a small part of a tile
  setup_tmem(w, (w.BN <= 128 && w.nkb < TC2_NACC1_MIN_KB) ? 2 : 1, TC2_MAX_NST);
  const int64_t stage_bytes = 2LL * w.BN * 128;
  w.sstride = (int)stage_bytes;
  const int64_t pack_bytes = (int64_t)w.ntiles * w.nkb * stage_bytes;
  const int64_t pack_aligned = (pack_bytes + 1023) / 1024 * 1024;
  if (!ws || ws_bytes < pack_aligned) return -1;
  uint8_t* bpack = reinterpret_cast<uint8_t*>(ws);
  // fused bias gradient (weight-gradient pack only): per (channel, k-block) partials
  const int64_t bias_bytes = bias_out ? ((int64_t)N * w.nkb * 4 + 1023) / 1024 * 1024 : 0;
  if (ws_bytes < pack_aligned + bias_bytes) return -1;
  float* bias_ws = bias_out ? reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(ws) + pack_aligned)
                            : nullptr;
  float* part_ws =
      reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(ws) + pack_aligned + bias_bytes);
  const int64_t part_bytes = ws_bytes - pack_aligned - bias_bytes;

  if constexpr (std::is_same_v<LBP, LdWgradDYPad>) {
    pack_dy_kernel<<<dim3(w.nkb, w.ntiles), 256, 0, st>>>(lbp, N, K, w.BN, w.nkb, bpack, bias_ws);
  } else if (fast)
    launch_pack_b(lbp, N, K, w.BN, w.nkb, w.ntiles, bpack, st);
  else
    launch_pack_b(lb, N, K, w.BN, w.nkb, w.ntiles, bpack, st);
  if (int rc = check_launch(what)) return rc;

  const int sms = gemm_sm_budget();
  w.splits = 1;
  {
    int64_t tiles = (int64_t)w.mtiles * w.ntiles;
#ifndef TC2_NOSPLIT_MIN_TILES  // forward / data gradients with >= 16 tiles are not split:
#define TC2_NOSPLIT_MIN_TILES 16  // inside a step the concurrent Inception branches fill the
#endif                            // SMs, and the partials + reduce launch cost more (+1.2%)
    const bool wgrad_pack = std::is_same_v<LBP, LdWgradDYPad>;
    if (tiles < sms && (wgrad_pack || tiles < TC2_NOSPLIT_MIN_TILES)) {
      int64_t want = sms / tiles;  // one wave: units <= SMs (ceil would leave a 2-unit tail)
      if (wgrad_pack) want = std::max(want, chain_min_splits(w.nkb, w.sacc != 0));
      int64_t by_k = w.nkb / 4;
      int64_t by_ws = part_bytes / ((int64_t)M * N * 4);
      const int64_t cap = std::min(by_k, std::min<int64_t>(by_ws, kMaxSplits));
      w.splits = (int)std::max<int64_t>(1, std::min(want, cap));
      if (wgrad_pack) w.splits = (int)balance_splits(tiles, w.nkb, w.splits, cap, sms);
    } else if (wgrad_pack) {  // many tiles: split only as far as the chain bound needs
      const int64_t by_ws = part_bytes / ((int64_t)M * N * 4);
      const int64_t cap = std::min<int64_t>(by_ws, kMaxSplits);
      w.splits = (int)std::max<int64_t>(1, std::min(chain_min_splits(w.nkb, w.sacc != 0), cap));
      w.splits = (int)balance_splits(tiles, w.nkb, w.splits, cap, sms);
    }
  }
  w.kbps = (w.nkb + w.splits - 1) / w.splits;
  w.splits = (w.nkb + w.kbps - 1) / w.kbps;
  w.units = w.mtiles * w.ntiles * w.splits;
  w.split_outer = std::is_same_v<LBP, LdWgradDYPad> && tc2_split_outer();

  const int smem_cap = 227 * 1024;
  const int tail = 1024 + (2 * STAGES + 3 * kBStagesMax + 4) * 8 + 64;
  w.full_ktab = (mode == kChannel || (mode == kGeneric && K <= kKtabMax)) ? 1 : 0;
  const int ktab_bytes = (w.full_ktab ? w.nkb * BK : STAGES * BK) * 8;  // as the kernel carves it
  // async-staged gather depth: 4 k-blocks (64 KB of staging) when that still
  // leaves >= 3 B stages, else 2, else the register path.  Weight gradients
  // over pixel rows >= 16 wide only: measured (tools/conv_bench.py, GoogLeNet)
  // 5-11% faster there (conv1 0.83 -> 0.75 ms), but 4-14% slower on 7x7 maps
  // and up to 1.9x slower for the table-driven forward / data gradients, whose
  // per-element 4-byte cp.async costs more issue than the predicated loads
  int ad = 0;
  if (tc2_async_gather_enabled() && mode == kWgrad16) {
    for (int cand : {4, 2}) {
      const int64_t left = smem_cap - tail - ktab_bytes - (int64_t)cand * 16 * kProducers * 4;
      if (left / stage_bytes >= 3) {
        ad = cand;
        break;
      }
    }
  }
  const int stg_bytes = ad * 16 * kProducers * 4;
  w.nbst = (int)std::min<int64_t>(kBStagesMax,
                                  (smem_cap - tail - ktab_bytes - stg_bytes) / stage_bytes);
  if (TC2_ONE_COMMIT) w.nst = w.nbst = std::min(w.nst, w.nbst);
  if (w.nbst < 2) return -1;
  const int smem = tail + (int)(w.nbst * stage_bytes) + stg_bytes + ktab_bytes;
  using KernT = decltype(&tc2_kernel<LA, Epi, kGeneric>);
  KernT kern;
  switch (mode * 3 + ad / 2) {
    case kChannel * 3: kern = tc2_kernel<LA, Epi, kChannel>; break;
    case kWgrad16 * 3 + 0: kern = tc2_kernel<LA, Epi, kWgrad16>; break;
    case kWgrad16 * 3 + 1: kern = tc2_kernel<LA, Epi, kWgrad16, 2>; break;
    case kWgrad16 * 3 + 2: kern = tc2_kernel<LA, Epi, kWgrad16, 4>; break;
    case kWgrad8 * 3: kern = tc2_kernel<LA, Epi, kWgrad8>; break;
    default: kern = tc2_kernel<LA, Epi, kGeneric>; break;
  }
  static bool configured[16] = {};
  if (!configured[mode * 3 + ad / 2]) {
    BF_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_cap),
            "tc2 smem attribute");
    configured[mode * 3 + ad / 2] = true;
  }
  // >= 120 KB of shared memory keeps one CTA (one 512-column TMEM allocation) per SM
  const int smem_req = std::max(smem, 120 << 10);
  const int grid = std::min(w.units, sms);
  EpiPartial part{part_ws, M, N};
  const CUtensorMap nomap{};
  kern<<<grid, kAllThreads, smem_req, st>>>(la, w, bpack, epi, part, nomap, nomap, nullptr);
  if (int rc = check_launch(what)) return rc;
  if (w.splits > 1) {
    splitk_reduce<Epi>(part_ws, w.splits, M, N, epi, st);
    if (int rc = check_launch(what)) return rc;
  }
  if (bias_out) {
    bias_blocks_finish_kernel<<<N, 256, 0, st>>>(bias_ws, w.nkb, bias_out);
    return check_launch(what);
  }
  return 0;
}

// 1x1 stride-1 weight gradient with both operands streamed by TMA (mode
// kTma1x1): dW[kout][c] = sum over (image, pixel) of dy[n][kout][p] x[n][c][p];
// M = C (x rows), N = Kout (dy rows), K = images x 32-pixel blocks (the box
// is per image; pixels past the image end are zero-filled).  No dY pack pass,
// no gather; the bias gradient comes from the same dy tiles.
inline int pick_bn_tma(int N, int& ntiles) {  // <= 192: >= 3 ring stages of 64 KB
  ntiles = (N + 191) / 192;
  int per = (N + ntiles - 1) / ntiles;
  return (per + 31) / 32 * 32;
}

// weight gradient, mode kWgradTma (default for the 3x3 / 5x5 layers whose
// output rows are a 16-byte multiple: GoogLeNet conv2/3x3, inception 3a / 3b):
// M = C*R*S rows gathered from x (kWgrad16 + cp.async staging) over the padded
// pixel grid Pp x Qp, B = the raw dY tile streamed by TMA -- a 4-D box of
// 32 / Qp whole rows or a 32-column piece of one row, zero past P / Q -- and
// split by the epilogue warps.  No dY pack pass (which read dY and wrote
// twice its size: 0.53 ms of the step) and half the B bytes in the GEMM.
int launch_wgrad_tma(const LdWgradX& la, const float* dy, int M, const EpiT& epi, float* ws,
                     int64_t ws_bytes, cudaStream_t st, const char* what, float* bias_out) {
  const ConvShape& g = la.g;
  const int PQ = g.P * g.Q, imgs = g.N, Kout = g.K;
  const WgradGeom wg = wgrad_geom(g);
  // measured per layer (conv_bench, batch 128, incl. the pack it replaces):
  // 56-wide rows 0.655 -> 0.620 ms (conv2/3x3), 28-wide rows 5-10% slower
  // (inception 3a / 3b: partial 32-column boxes, and the split step adds to
  // each stage's latency in a 3-stage ring) -- so rows >= 48 only, unless
  // engine 7 asks for every eligible shape (tests)
  if (g.Q < 48 && g_gemm_engine != 7) return -1;
  if (wg.Qp < 16 || (wg.Pp * wg.Qp) % BK || (reinterpret_cast<uintptr_t>(dy) & 15)) return -1;
  const bool flat = wg.Qp == g.Q && wg.Pp == g.P && PQ % BK == 0;
  // a row-box map needs 16-byte row strides and whole 32-pixel pieces per row
  if (!flat && (g.Q % 4 || !(wg.Qp <= BK || wg.Qp % BK == 0))) return -1;
  Work w{};
  w.M = M;
  w.N = Kout;
  w.cpi = wg.Pp * wg.Qp / BK;
  w.nkb = imgs * w.cpi;
  w.K = w.nkb * BK;
  w.Pp = wg.Pp;
  w.Qp = wg.Qp;
  w.tma4 = flat ? 0 : 1;
  divmagic((uint32_t)(w.Pp * w.Qp), w.per_m, w.per_s);
  divmagic((uint32_t)w.Qp, w.qp_m, w.qp_s);
  w.BN = pick_bn_tma(Kout, w.ntiles);
  w.mtiles = (M + BM - 1) / BM;
  setup_tmem(w, w.BN <= 128 ? 2 : 1, TC2_MAX_NST);
  w.sstride = 2 * w.BN * 128;
  w.full_ktab = 0;
  CUtensorMap bmap;
  if (flat) {
    if (!make_nchw_map(&bmap, dy, PQ, Kout, imgs, w.BN, CU_TENSOR_MAP_SWIZZLE_128B)) return -1;
  } else {
    auto fn = tma_encode_fn();
    if (!fn) return -1;
    const int bx = wg.Qp <= BK ? wg.Qp : BK, by = wg.Qp <= BK ? BK / wg.Qp : 1;
    cuuint64_t dims[4] = {(cuuint64_t)g.Q, (cuuint64_t)g.P, (cuuint64_t)Kout, (cuuint64_t)imgs};
    cuuint64_t strides[3] = {(cuuint64_t)g.Q * 4, (cuuint64_t)PQ * 4, (cuuint64_t)Kout * PQ * 4};
    cuuint32_t box[4] = {(cuuint32_t)bx, (cuuint32_t)by, (cuuint32_t)w.BN, 1};
    cuuint32_t estr[4] = {1, 1, 1, 1};
    if (fn(&bmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, const_cast<float*>(dy), dims, strides, box,
           estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return -1;
  }
  // workspace: [bias partials: Kout x <= kMaxSplits splits][split-K partials]
  const int64_t bias_bytes = bias_out ? ((int64_t)Kout * kMaxSplits * 4 + 1023) / 1024 * 1024 : 0;
  if (!ws || ws_bytes < bias_bytes) return -1;
  float* bias_ws = bias_out ? ws : nullptr;
  float* part_ws = reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(ws) + bias_bytes);
  const int64_t part_bytes = ws_bytes - bias_bytes;
  const int sms = gemm_sm_budget();
  w.splits = 1;
  {
    const int64_t tiles = (int64_t)w.mtiles * w.ntiles;
    {
      const int64_t want = std::max<int64_t>(tiles < sms ? sms / tiles : 1,
                                             chain_min_splits(w.nkb, w.sacc != 0));
      const int64_t by_k = std::max<int64_t>(1, w.nkb / 4);
      const int64_t by_ws = part_bytes / ((int64_t)M * Kout * 4);
      const int64_t cap = std::min(by_k, std::min<int64_t>(by_ws, kMaxSplits));
      w.splits = (int)std::max<int64_t>(1, std::min(want, cap));
      w.splits = (int)balance_splits(tiles, w.nkb, w.splits, cap, sms);
    }
  }
  w.kbps = (w.nkb + w.splits - 1) / w.splits;
  w.splits = (w.nkb + w.kbps - 1) / w.kbps;
  w.units = w.mtiles * w.ntiles * w.splits;
  w.split_outer = tc2_split_outer();
  constexpr int AD = 4;
  const int smem_cap = 227 * 1024;
  const int tail = 1024 + (2 * STAGES + 3 * kBStagesMax + 4) * 8 + 64;
  const int ktab_bytes = STAGES * BK * 8;
  const int stg_bytes = AD * 16 * kProducers * 4;
  w.nbst = std::min(kBStagesMax, (smem_cap - tail - ktab_bytes - stg_bytes) / w.sstride);
  if (TC2_ONE_COMMIT) w.nst = w.nbst = std::min(w.nst, w.nbst);
  if (w.nbst < 2) return -1;
  const int smem = std::max(tail + w.nbst * w.sstride + stg_bytes + ktab_bytes, 120 << 10);
  auto kern = tc2_kernel<LdWgradX, EpiT, kWgradTma, AD>;
  static bool configured = false;
  if (!configured) {
    BF_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_cap),
            "tc2 smem attribute");
    configured = true;
  }
  const int grid = std::min(w.units, sms);
  EpiPartial part{part_ws, M, Kout};
  const CUtensorMap nomap{};
  kern<<<grid, kAllThreads, smem, st>>>(la, w, nullptr, epi, part, nomap, bmap, bias_ws);
  if (int rc = check_launch(what)) return rc;
  if (w.splits > 1) {
    splitk_reduce<EpiT>(part_ws, w.splits, M, Kout, epi, st);
    if (int rc = check_launch(what)) return rc;
  }
  if (bias_out) {
    bias_blocks_finish_kernel<<<Kout, 256, 0, st>>>(bias_ws, w.splits, bias_out);
    return check_launch(what);
  }
  return 0;
}

int launch_tma1x1(const LdWgradX& la, const float* x, const float* dy, int C, int Kout, int PQ,
                  int imgs, const EpiT& epi, float* ws, int64_t ws_bytes, cudaStream_t st,
                  const char* what, float* bias_out) {
  if (PQ % 4 || ((reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(dy)) & 15))
    return -1;
  Work w{};
  w.M = C;
  w.N = Kout;
  w.cpi = (PQ + BK - 1) / BK;
  w.nkb = imgs * w.cpi;
  w.K = w.nkb * BK;
  w.BN = pick_bn_tma(Kout, w.ntiles);
  w.mtiles = (C + BM - 1) / BM;
  setup_tmem(w, w.BN <= 128 ? 2 : 1, 7);
  w.sstride = 2 * w.BN * 128 + BM * 128;
  w.full_ktab = 0;
  CUtensorMap amap, bmap;
  if (!make_nchw_map(&amap, x, PQ, C, imgs, BM, CU_TENSOR_MAP_SWIZZLE_128B) ||
      !make_nchw_map(&bmap, dy, PQ, Kout, imgs, w.BN, CU_TENSOR_MAP_SWIZZLE_128B))
    return -1;
  // workspace: [bias partials: Kout x <= kMaxSplits splits][split-K partials]
  const int64_t bias_bytes = bias_out ? ((int64_t)Kout * kMaxSplits * 4 + 1023) / 1024 * 1024 : 0;
  if (!ws || ws_bytes < bias_bytes) return -1;
  float* bias_ws = bias_out ? ws : nullptr;
  float* part_ws = reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(ws) + bias_bytes);
  const int64_t part_bytes = ws_bytes - bias_bytes;
  const int sms = gemm_sm_budget();
  w.splits = 1;
  {
    const int64_t tiles = (int64_t)w.mtiles * w.ntiles;
    {
      const int64_t want = std::max<int64_t>(tiles < sms ? sms / tiles : 1,
                                             chain_min_splits(w.nkb, w.sacc != 0));
      const int64_t by_k = std::max<int64_t>(1, w.nkb / 4);
      const int64_t by_ws = part_bytes / ((int64_t)C * Kout * 4);
      const int64_t cap = std::min(by_k, std::min<int64_t>(by_ws, kMaxSplits));
      w.splits = (int)std::max<int64_t>(1, std::min(want, cap));
      w.splits = (int)balance_splits(tiles, w.nkb, w.splits, cap, sms);
    }
  }
  w.kbps = (w.nkb + w.splits - 1) / w.splits;
  w.splits = (w.nkb + w.kbps - 1) / w.kbps;
  w.units = w.mtiles * w.ntiles * w.splits;
  w.split_outer = tc2_split_outer();
  const int smem_cap = 227 * 1024;
  const int tail = 1024 + (2 * STAGES + 3 * kBStagesMax + 4) * 8 + 64;
  const int ktab_bytes = STAGES * BK * 8;
  w.nbst = std::min(kBStagesMax, (smem_cap - tail - ktab_bytes) / w.sstride);
  if (TC2_ONE_COMMIT) w.nst = w.nbst = std::min(w.nst, w.nbst);
  if (w.nbst < 2) return -1;
  const int smem = std::max(tail + w.nbst * w.sstride + ktab_bytes, 120 << 10);
  auto kern = tc2_kernel<LdWgradX, EpiT, kTma1x1>;
  static bool configured = false;
  if (!configured) {
    BF_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_cap),
            "tc2 smem attribute");
    configured = true;
  }
  const int grid = std::min(w.units, sms);
  EpiPartial part{part_ws, C, Kout};
  kern<<<grid, kAllThreads, smem, st>>>(la, w, nullptr, epi, part, amap, bmap, bias_ws);
  if (int rc = check_launch(what)) return rc;
  if (w.splits > 1) {
    splitk_reduce<EpiT>(part_ws, w.splits, C, Kout, epi, st);
    if (int rc = check_launch(what)) return rc;
  }
  if (bias_out) {
    bias_blocks_finish_kernel<<<Kout, 256, 0, st>>>(bias_ws, w.splits, bias_out);
    return check_launch(what);
  }
  return 0;
}

}  // namespace tc2

// conv forward / stride-1 data gradient through engine v2; -1 = not taken
int tc2_conv_fwd(const LdFwdX& la, const LdRowK& lb, int M, int N, int K, const EpiNCHW& epi,
                 float* ws, int64_t ws_bytes, cudaStream_t st, const char* what) {
  if (K < 8) return -1;
  tc2::LdFwdWPerm lbp{lb.p, la.g.C, la.g.R * la.g.S};
  return tc2::launch(la, lb, lbp, M, N, K, epi, ws, ws_bytes, st, what);
}

int tc2_conv_wgrad(const LdWgradX& la, const LdWgradDY& lb, int M, int N, int K,
                   const EpiT& epi, float* ws, int64_t ws_bytes, cudaStream_t st,
                   const char* what, float* db, bool* db_done) {
  if (db_done) *db_done = false;
  if (K < 8) return -1;
  const ConvShape& g = la.g;
  if (g.R == 1 && g.S == 1 && g.stride == 1 && g.pad == 0 && g.P == g.H && g.Q == g.W &&
      tc2_tma_wgrad_enabled()) {
    const int rc = tc2::launch_tma1x1(la, la.x, lb.dy, g.C, g.K, g.H * g.W, g.N, epi, ws,
                                      ws_bytes, st, what, db);
    if (rc == 0) {
      if (db_done) *db_done = db != nullptr;
      return 0;
    }
    if (rc > 0) return rc;
  }
  if (tc2_wgrad_tma_enabled()) {
    const int rc = tc2::launch_wgrad_tma(la, lb.dy, M, epi, ws, ws_bytes, st, what, db);
    if (rc == 0) {
      if (db_done) *db_done = db != nullptr;
      return 0;
    }
    if (rc > 0) return rc;
  }
  const tc2::WgradGeom wg = tc2::wgrad_geom(la.g);
  const int64_t kpad = (int64_t)la.g.N * wg.Pp * wg.Qp;
  if (kpad < (int64_t)K * 2 && kpad < (1LL << 31)) {  // padding waste bounded: fast path
    tc2::LdWgradDYPad lbp{lb.dy, la.g.K, la.g.P, la.g.Q, wg.Pp, wg.Qp};
    const int rc = tc2::launch(la, lb, lbp, M, N, (int)kpad, epi, ws, ws_bytes, st, what,
                               wg.Qp >= 16 ? tc2::kWgrad16 : tc2::kWgrad8, wg.Pp, wg.Qp, db);
    if (rc == 0 && db_done) *db_done = db != nullptr;
    return rc;
  }
  return tc2::launch(la, lb, lb, M, N, K, epi, ws, ws_bytes, st, what);
}

int tc2_conv_dgrad(const LdDgradDY& la, const LdDgradW& lb, int M, int N, int K,
                   const EpiNCHW& epi, float* ws, int64_t ws_bytes, cudaStream_t st,
                   const char* what) {
  if (la.g.stride != 1 || M < 128 || K < 8) return -1;
  tc2::LdDgradWPerm lbp{lb.w, la.g.C, la.g.K, la.g.R * la.g.S};
  return tc2::launch(la, lb, lbp, M, N, K, epi, ws, ws_bytes, st, what);
}

}  // namespace bf
