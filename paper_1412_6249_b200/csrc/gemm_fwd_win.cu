// tcgen05 engine "fwd-win": the forward of a convolution over few input
// channels (GoogLeNet conv1: 3 -> 64, 7x7 stride 2, 224 -> 112).
//
//   y[n][k][p][q] = b[k] + sum_{c,r,s} w[k][c][r][s] * x[n][c][st*p + r - pad][st*q + s - pad]
//
// Engine v2 gathers the stride-2 im2col element by element from global memory
// through per-row index tables (0.342 ms for conv1 at batch 128, producer-
// bound at ~88 TFLOP/s).  Here one tile is 128 output pixels of ONE output row
// (img, p, q0..q0+127), and for each input row (c, r) the S taps of all 128
// pixels lie in one contiguous window of st*127 + S floats:
// * the C*R windows of a tile are staged by 16-byte cp.async spread over all
//   producer threads, kWinSlots-1 tiles ahead, zero-filled outside the image
//   (x rows are read ~R/st times, from L2);
// * A = the im2col rows, one TMEM lane per output pixel.  The contraction is
//   laid out in groups of 8 columns per (c, r) (taps s < S, zeros after), so a
//   32-column k-block is 4 windows; thread j reads window[st*j + s] for s < S
//   at compile-time offsets (S and the stride are template parameters) and
//   writes the big part (x as is) and the RN-adjusted small part into a TMEM
//   ring (tcgen05.st).  The four producer warps of a lane quarter take
//   alternate k-blocks, so four stages fill concurrently;
// * B = the weights, packed once per launch (pack_b_kernel: big/small halves,
//   128B-swizzled, K-major) and resident in shared memory for the whole
//   persistent CTA;
// * 3xTF32 with a separate small-term accumulator: per k-step one N = 2K MMA
//   A_big * [B_big | B_small] and one N = K MMA A_small * B_big accumulating
//   into the small half; the epilogue adds the halves in fp32 RN (gemm_tc2.cu);
// * double-buffered accumulators: tile t's epilogue (bias, the fused ReLU,
//   NCHW stores through EpiNCHW) overlaps tile t+1's MMAs.
// Per tile the contraction is C*R*8 (168, padded to 192) deep: far below the
// round-toward-zero chain bound, no split.
//
// Measured (conv1, batch 128, y stored): 0.28 ms vs engine v2's 0.342.  What
// bounds it: with the windows and stores taken out it still runs 0.20 ms
// against ~0.11 ms of MMA issue -- the commit -> mbarrier -> producer round
// trip (~3000 cycles, profiles/r01_mma_probe.md) exceeds what the TMEM A ring
// can buffer at N = 64 (four stages x ~360 cycles); six stages without the
// separate small accumulator (FWIN_SACC=0) measure the same.  Rejected
// variants: a per-column offset table with 8 producer warps (0.36 ms, ~10
// issue slots per value); window staging by a single loader warp (cp.async:
// 0.69 ms) or by cp.async.bulk per window (0.53 ms) -- their issue is serial;
// TMA tiled 4-D boxes of the rows faulted: a TMA box's innermost start must
// be a 16-byte multiple (tools/tma4d_probe.cu), the window start st*q0 - pad
// is not -- an aligned start with the offset applied by the producers would
// work, but the window staging is not what bounds this kernel.
#include <stdlib.h>

#include <algorithm>

#include "gemm_common.cuh"
#include "gemm_engines.cuh"
#include "tc_ptx.cuh"

namespace bf {
namespace fwin {

using namespace tcu;

constexpr int BK = 32;
#ifndef FWIN_SACC
#define FWIN_SACC 1
#endif
// with the separate small-term accumulator an accumulator buffer is 2K
// columns (two buffers + four A stages fill TMEM for K = 64); without it, K
// columns and six A stages
constexpr int kStages = FWIN_SACC ? 4 : 6;  // TMEM A ring stages (64 columns: 32 big + 32 small)
constexpr int kAccMul = FWIN_SACC ? 2 : 1;
constexpr int kWinSlots = 3; // window staging ring: cp.async kWinSlots-1 tiles ahead
constexpr int kMaxKb = 8;    // C*R <= 32 windows
// warps: 0 loads (weights, windows), 1 MMA (+ TMEM allocation), 2-17
// producers (four per TMEM lane quarter: warp g writes A stage g), 18-21
// epilogue (one per lane quarter)
constexpr int kLoadWarp = 0, kMmaWarp = 1, kProdWarp0 = 2, kProdWarps = 16;
constexpr int kEpiWarp0 = kProdWarp0 + kProdWarps, kEpiWarps = 4;
constexpr int kThreads = (kEpiWarp0 + kEpiWarps) * 32;
constexpr int kProducers = kProdWarps * 32;
constexpr int kMaxIds = 3;  // window chunks per producer thread: C*R*nch <= 1536
constexpr int kOwners = kProdWarps / 4;  // producer warps per lane quarter

struct Geo {
  int N, C, H, W, K, R, S, P, Q, st, pad;
  int CR, CRS, nkb;     // windows, taps, k-blocks (8 columns per window, 4 windows per k-block)
  int nqt, tiles;       // 128-pixel tiles per output row, total tiles
  int win_floats;       // staged floats per window (16-byte multiple)
  int kimg;             // bytes of one k-block's B image: [big K rows | small K rows] x 128B
  int abase;            // first TMEM column of the A ring (after 2 x 2K accumulator columns)
  uint64_t pi_m, nq_m;  // multiply-shift constants: x / (P*nqt), x / nqt
  int pi_s, nq_s;
};

// m = ceil(2^(31+l) / d), l = ceil(log2 d): exact x / d for every x < 2^31
inline void fwin_divmagic(uint32_t d, uint64_t& m, int& s) {
  int l = 0;
  while ((1ull << l) < d) ++l;
  s = 31 + l;
  m = ((1ull << s) + d - 1) / d;
}


// B operand column k = 8*(c*R + r) + s: w[n][c][r][s] for s < S, else 0
struct LdW8 {
  static constexpr bool kMContig = false;
  const float* w;
  int S, CRS;
  __device__ __forceinline__ float operator()(int n, int k) const {
    const int cr = k >> 3, s = k & 7;
    return (s < S && cr * S + s < CRS) ? w[(int64_t)n * CRS + cr * S + s] : 0.f;
  }
};

__device__ __forceinline__ void tmem_st8(uint32_t taddr, const float (&v)[8]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(taddr),
      "f"(v[0]), "f"(v[1]), "f"(v[2]), "f"(v[3]), "f"(v[4]), "f"(v[5]), "f"(v[6]), "f"(v[7])
      : "memory");
}
__device__ __forceinline__ float lds_f32(uint32_t a) {
  float v;
  asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(a));
  return v;
}

template <int S_, int ST_>
__global__ void __launch_bounds__(kThreads, 1)
    fwin_kernel(const float* __restrict__ x, const uint8_t* __restrict__ bpack, Geo g,
                EpiNCHW epi) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint8_t* bsm = base;                                        // nkb B images
  float* staging = reinterpret_cast<float*>(bsm + g.nkb * g.kimg);
  uint64_t* bars = reinterpret_cast<uint64_t*>(staging + kWinSlots * g.CR * g.win_floats);
  uint64_t* b_full = bars;               // the resident weights landed
  uint64_t* a_full = b_full + 1;         // producers wrote A big / small (stage)
  uint64_t* empty = a_full + kStages;    // MMAs of the stage done
  uint64_t* acc_full = empty + kStages;  // [2]
  uint64_t* acc_empty = acc_full + 2;    // [2]
  uint64_t* win_full = acc_empty + 2;    // [kWinSlots] the tile's windows landed
  uint64_t* win_empty = win_full + kWinSlots;  // [kWinSlots] producers done reading them
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(win_empty + kWinSlots);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int K = g.K;

  if (warp == kMmaWarp) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
        smem_u32(tmem_slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (threadIdx.x == 0) {
    mbar_init(b_full, 1);
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&a_full[s], 4);  // one elected arrival per lane-quarter warp owning the stage
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&acc_full[b], 1);
      mbar_init(&acc_empty[b], kEpiWarps * 32);
    }
    for (int w = 0; w < kWinSlots; ++w) {
      mbar_init(&win_full[w], kProducers);  // each producer's cp.async completions
      mbar_init(&win_empty[w], kProdWarps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  // tile u -> (image, output row, 128-pixel block): multiply-shift divisions
  // (exact for u < 2^31; the host checks), no integer-division sequences
  auto tile_coords = [&](int u, int& img, int& p, int& q0) {
    const int per_img = g.P * g.nqt;
    img = (int)(((uint64_t)(uint32_t)u * g.pi_m) >> g.pi_s);
    const int rem = u - img * per_img;
    p = (int)(((uint64_t)(uint32_t)rem * g.nq_m) >> g.nq_s);
    q0 = (rem - p * g.nqt) * BM;
  };

  if (warp == kLoadWarp) {
    // ======================= resident weights (once) =======================
    if (blockIdx.x < g.tiles) {
      if (lane == 0) {
        mbar_arrive_expect_tx(b_full, (uint32_t)(g.nkb * g.kimg));
        for (int kb = 0; kb < g.nkb; ++kb)
          bulk_g2s(smem_u32(bsm + kb * g.kimg), bpack + (size_t)kb * g.kimg, (uint32_t)g.kimg,
                   b_full);
      }
    }
    __syncwarp();
  } else if (warp == kMmaWarp) {
    // ======================= MMA issuer =======================
    const uint32_t idesc2 = tf32_idesc(2 * K), idesc1 = tf32_idesc(K);
    if (blockIdx.x < g.tiles) mbar_wait(b_full, 0);
    int s = 0, local = 0;
    uint32_t ph = 0;
    for (int u = blockIdx.x; u < g.tiles; u += gridDim.x, ++local) {
      const int buf = local & 1;
      mbar_wait(&acc_empty[buf], ((local >> 1) & 1) ^ 1);
      tc_fence_after();
      const uint32_t d = tmem + (uint32_t)(buf * kAccMul * K), dsm = d + (uint32_t)K;
      for (int kb = 0; kb < g.nkb; ++kb) {
        mbar_wait(&a_full[s], ph);
        tc_fence_after();
        const uint64_t bb = sw128_desc(smem_u32(bsm + kb * g.kimg));
        const uint32_t ab = tmem + (uint32_t)(g.abase + s * 64), as = ab + 32;
        if (!FWIN_SACC && elect_one()) {
          const uint64_t bs = bb + (uint64_t)((K * 128) >> 4);
#pragma unroll
          for (int ks = 0; ks < BK / 8; ++ks) {
            const uint64_t k2 = (uint64_t)((ks * 32) >> 4);
            if (ks == 0 && kb == 0)
              mma_ts_flag<0>(d, ab, bb, idesc1);
            else
              mma_ts_flag<1>(d, ab + ks * 8, bb + k2, idesc1);
            mma_ts_flag<1>(d, ab + ks * 8, bs + k2, idesc1);
            mma_ts_flag<1>(d, as + ks * 8, bb + k2, idesc1);
          }
          tc_commit(&empty[s]);
        } else if (FWIN_SACC && elect_one()) {
          if (kb == 0)
            mma_ts_flag<0>(d, ab, bb, idesc2);
          else
            mma_ts_flag<1>(d, ab, bb, idesc2);
          mma_ts_flag<1>(dsm, as, bb, idesc1);
#pragma unroll
          for (int ks = 1; ks < BK / 8; ++ks) {
            const uint64_t k2 = (uint64_t)((ks * 32) >> 4);
            mma_ts_flag<1>(d, ab + ks * 8, bb + k2, idesc2);
            mma_ts_flag<1>(dsm, as + ks * 8, bb + k2, idesc1);
          }
          tc_commit(&empty[s]);
        }
        __syncwarp();
        if (++s == kStages) {
          s = 0;
          ph ^= 1;
        }
      }
      if (elect_one()) tc_commit(&acc_full[buf]);
      __syncwarp();
    }
  } else if (warp < kEpiWarp0) {
    // ======================= producers: windows -> A (TMEM) =======================
    // warp g of a lane quarter owns A stage g: it writes all 32 columns (4
    // windows) of every k-block k with k = g mod 4 (k counted over the CTA's
    // whole tile sequence), so the four warps of a quarter fill four stages
    // concurrently (one warp per k-block would serialise on its latency)
    const int quarter = warp & 3, gst = (warp - kProdWarp0) >> 2;
    const int j = quarter * 32 + lane;  // TMEM lane = pixel q0 + j of the tile
    const uint32_t la = tmem + ((uint32_t)(quarter * 32) << 16) + (uint32_t)g.abase;
    const uint32_t stg0 = smem_u32(staging);
    const int wf = g.win_floats;
    // window staging: a window is the 16-byte aligned row segment
    // [(st*q0 - pad) & ~3, +win_floats) of x row (img, c, st*p + r - pad); its
    // 16-byte chunks are spread over all producer threads (cp.async, zero
    // fill outside the image), kWinSlots-1 tiles ahead, each thread's
    // completions arriving on the slot's win_full.  (One loader warp issuing
    // them, or a few cp.async.bulk copies per window, measured 2-2.5x slower:
    // the issue is serial.)
    const int t = (warp - kProdWarp0) * 32 + lane;
    const int nch = wf / 4;
    // chunk i of this thread: (c, r, f) packed as c << 24 | r << 16 | f
    int id_crf[kMaxIds], nid = 0;
    for (int id = t; id < g.CR * nch && nid < kMaxIds; id += kProducers, ++nid) {
      const int cr = id / nch, f = id - cr * nch, c = cr / g.R;
      id_crf[nid] = (c << 24) | ((cr - c * g.R) << 16) | f;
    }
    auto issue = [&](int u, int slot, uint32_t eph) {
      if (u >= g.tiles) return;
      mbar_wait(&win_empty[slot], eph);
      int img, p, q0;
      tile_coords(u, img, p, q0);
      const int a0 = (ST_ * q0 - g.pad) & ~3;
      const uint32_t sbase = stg0 + (uint32_t)(slot * g.CR * wf * 4);
#pragma unroll
      for (int i = 0; i < kMaxIds; ++i) {
        if (i < nid) {
          const int c = id_crf[i] >> 24, r = (id_crf[i] >> 16) & 0xff, f = id_crf[i] & 0xffff;
          const int ih = ST_ * p + r - g.pad, iw = a0 + 4 * f;
          const bool ok = (unsigned)ih < (unsigned)g.H && iw >= 0 && iw < g.W;
          const float* src = ok ? x + (((int64_t)img * g.C + c) * g.H + ih) * g.W + iw : x;
          const uint32_t dst = sbase + (uint32_t)(((c * g.R + r) * wf + 4 * f) * 4);
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst),
                       "l"(src), "r"(ok ? 16 : 0)
                       : "memory");
        }
      }
      asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(
                       smem_u32(&win_full[slot]))
                   : "memory");
    };
    // tiles blockIdx.x + i*gridDim.x, i = 0, 1, ...: tile i uses slot i % kWinSlots
    // with win_full parity (i / kWinSlots) & 1
    for (int i = 0; i < kWinSlots - 1; ++i) issue(blockIdx.x + i * gridDim.x, i, 1);
    int slot = 0, kfirst = gst;  // kfirst: this warp's first k-block in the tile
    int gkb0 = 0;                // CTA-wide index of the tile's first k-block
    int ahead = kWinSlots - 1;             // next tile index to stage
    uint32_t wph = 0;
    for (int u = blockIdx.x; u < g.tiles; u += gridDim.x) {
      issue(blockIdx.x + ahead * gridDim.x, ahead % kWinSlots,
            ((ahead / kWinSlots) & 1) ^ 1);
      ++ahead;
      mbar_wait(&win_full[slot], wph);
      int img, p, q0;
      tile_coords(u, img, p, q0);
      const int o = (ST_ * q0 - g.pad) - ((ST_ * q0 - g.pad) & ~3);
      // shared-space address (32-bit) of this lane's first tap in window 0
      const uint32_t wa0 = stg0 + (uint32_t)((slot * g.CR * wf + o + ST_ * j) * 4);
      int kb = kfirst;
#pragma unroll 1
      for (; kb < g.nkb; kb += kOwners) {
        const int gkb = gkb0 + kb;
        const int st = gkb % kStages;
        mbar_wait(&empty[st], ((gkb / kStages) & 1) ^ 1);
        tc_fence_after();
        const uint32_t lst = la + (uint32_t)(64 * st);
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          float big[16], small[16];
#pragma unroll
          for (int w2 = 0; w2 < 2; ++w2) {
            const int cr = 4 * kb + 2 * h + w2;
            const uint32_t wa = wa0 + (uint32_t)(cr * wf * 4);
            const bool ok = cr < g.CR;
#pragma unroll
            for (int e = 0; e < 8; ++e)
              big[8 * w2 + e] = (e < S_ && ok)
                                    ? lds_f32(wa + 4 * e)
                                    : 0.f;
          }
#pragma unroll
          for (int e = 0; e < 16; ++e) small[e] = tf32_small(big[e]);
          tmem_st16(lst + 16 * h, big);
          tmem_st16(lst + 32 + 16 * h, small);
        }
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&a_full[st]);
      }
      kfirst = kb - g.nkb;  // carries into the next tile's k-blocks
      gkb0 += g.nkb;
      // every window value of the tile is in registers / TMEM by now
      __syncwarp();
      if (lane == 0) mbar_arrive(&win_empty[slot]);
      if (++slot == kWinSlots) {
        slot = 0;
        wph ^= 1;
      }
    }
  } else {
    // ======================= epilogue =======================
    const int quarter = warp & 3;
    const int j = quarter * 32 + lane;
    const uint32_t taddr = tmem + ((uint32_t)(quarter * 32) << 16);
    int local = 0;
    for (int u = blockIdx.x; u < g.tiles; u += gridDim.x, ++local) {
      const int buf = local & 1;
      mbar_wait(&acc_full[buf], (local >> 1) & 1);
      tc_fence_after();
      int img, p, q0;
      tile_coords(u, img, p, q0);
      const bool live = q0 + j < g.Q;
      const RowPtr rp = live ? epi.row((img * g.P + p) * g.Q + q0 + j) : RowPtr{nullptr, 0.f};
      const uint32_t d = taddr + (uint32_t)(buf * kAccMul * K);
#pragma unroll 1
      for (int c0 = 0; c0 < K; c0 += 16) {
        uint32_t v[16];
        tmem_ld16(d + (uint32_t)c0, v);
        if (FWIN_SACC) {
          uint32_t sv[16];
          tmem_ld16(d + (uint32_t)(K + c0), sv);
#pragma unroll
          for (int e = 0; e < 16; ++e)
            v[e] = __float_as_uint(__fadd_rn(__uint_as_float(v[e]), __uint_as_float(sv[e])));
        }
        if (live) epi.store16(rp, c0, v, K - c0);
      }
      tc_fence_before();
      mbar_arrive(&acc_empty[buf]);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == kMmaWarp) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
  }
}

}  // namespace fwin

bool fwd_win_enabled() {
  const char* e = getenv("PURINE_B200_FWD_WIN");
  return !(e && *e && atoi(e) == 0);
}

// -1 when the shape is not taken
int fwd_win_conv(const ConvShape& g, const float* x, const float* w, const EpiNCHW& epi,
                 float* ws, int64_t ws_bytes, cudaStream_t st, const char* what) {
  using namespace fwin;
  if (!fwd_win_enabled()) return -1;
  const int CRS = g.C * g.R * g.S;
  if (g.K > 64 || g.K < 16 || g.K % 16 || g.C * g.R > kMaxKb * 4 || g.S > 8 || g.W % 4 ||
      (reinterpret_cast<uintptr_t>(x) & 15))
    return -1;
  int variant = -1;
  {
    const int tbl[6][2] = {{7, 2}, {5, 2}, {3, 2}, {7, 1}, {5, 1}, {3, 1}};
    for (int i = 0; i < 6; ++i)
      if (g.S == tbl[i][0] && g.stride == tbl[i][1]) variant = i;
  }
  if (variant < 0) return -1;
  Geo q{};
  q.N = g.N; q.C = g.C; q.H = g.H; q.W = g.W; q.K = g.K; q.R = g.R; q.S = g.S;
  q.P = g.P; q.Q = g.Q; q.st = g.stride; q.pad = g.pad;
  q.CR = g.C * g.R;
  q.CRS = CRS;
  q.nkb = (q.CR + 3) / 4;
  q.nqt = (g.Q + BM - 1) / BM;
  const int64_t tiles = (int64_t)g.N * g.P * q.nqt;
  if (tiles > (1LL << 30)) return -1;
  q.tiles = (int)tiles;
  fwin_divmagic((uint32_t)(q.P * q.nqt), q.pi_m, q.pi_s);
  fwin_divmagic((uint32_t)q.nqt, q.nq_m, q.nq_s);
  q.win_floats = (3 + g.stride * (BM - 1) + g.S + 3) / 4 * 4;
  q.kimg = 2 * g.K * 128;
  q.abase = (2 * kAccMul * g.K + 63) / 64 * 64;
  if (q.abase + kStages * 64 > 512 || q.CR * (q.win_floats / 4) > kMaxIds * kProducers) return -1;
  const int smem_cap = 227 * 1024;
  const int smem = 1024 + q.nkb * q.kimg + kWinSlots * q.CR * q.win_floats * 4 +
                   (1 + 2 * kStages + 4 + 2 * kWinSlots) * 8 + 16;
  if (smem > smem_cap) return -1;
  const int64_t pack_bytes = (int64_t)q.nkb * q.kimg;
  if (!ws || ws_bytes < pack_bytes) return -1;
  uint8_t* bpack = reinterpret_cast<uint8_t*>(ws);
  launch_pack_b(LdW8{w, g.S, CRS}, g.K, q.nkb * BK, g.K, q.nkb, 1, bpack, st);
  if (int rc = check_launch(what)) return rc;
  const int grid = (int)std::min<int64_t>(tiles, gemm_sm_budget());
#define FWIN_LAUNCH(I, SS, TT)                                                              \
  case I:                                                                                   \
    BF_CUDA(cudaFuncSetAttribute(fwin_kernel<SS, TT>,                                       \
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, smem_cap),    \
            "fwd-win smem attribute");                                                      \
    fwin_kernel<SS, TT><<<grid, kThreads, smem, st>>>(x, bpack, q, epi);                 \
    break;
  switch (variant) {
    FWIN_LAUNCH(0, 7, 2)
    FWIN_LAUNCH(1, 5, 2)
    FWIN_LAUNCH(2, 3, 2)
    FWIN_LAUNCH(3, 7, 1)
    FWIN_LAUNCH(4, 5, 1)
    FWIN_LAUNCH(5, 3, 1)
  }
#undef FWIN_LAUNCH
  return check_launch(what);
}

}  // namespace bf
