// tcgen05 engine "wgrad-T": the weight gradient of a convolution over few
// input channels (GoogLeNet conv1: 3 -> 64, 7x7 stride 2), computed
// transposed.
//
//   dW[kout][c,r,s] = sum_{n,p,q} dY[n][kout][p][q] * X[n][c][st*p + r - pad][st*q + s - pad]
//
// Engine v2 takes rows = (c, r, s) (147 for conv1: two 128-row M tiles, the
// second 15% full) and gathers the stride-2 im2col operand element by
// element; it is producer-bound at 40 TFLOP/s.  Here the MMA is
//   D[m = kout][n = (c, r, s)] = A[kout][pixels] x B[(c, r, s)][pixels]^T
// * A = dY: a TMA box {32 q, 1 p, Kout rows} straight from NCHW (K-major,
//   128B swizzle) -- no gather; rows Kout..127 of the 128-row M tile stay zero
//   (an M = 64 MMA costs as much as M = 128, B300_MICROARCH tcgen05 floor);
// * B = the im2col of x: for a k-block of 32 output pixels on one output row
//   and one input row (c, r), the S taps of all 32 pixels lie in ONE
//   contiguous window of st*31 + S floats (69 for conv1) -- staged by 16-byte
//   cp.async per (c, r) window, then each lane j writes its S taps
//   window[o + st*j + s] into rows (c, r, s) of the swizzled B image (big and
//   small part).  Per k-block: C*R*S*32 gathered elements from C*R windows,
//   against 2 x 128 x 32 per-element table gathers before.
// * 3xTF32 with separate big / small accumulators (A_big*B_big into columns
//   [0, NP), A_big*B_small + A_small*B_big into [NP, 2NP)), added in fp32 RN
//   by the epilogue (see gemm_tc2.cu).
// K (pixels) is split into units of at most max_chain_kb() k-blocks (the
// round-toward-zero accumulation bound, gemm_common.cuh); partials are summed
// by the split-K reduction; the bias gradient comes from the same dY tiles.
// Pixel k-blocks never straddle output rows: each output row is ceil(Q/32)
// k-blocks, the pixels past Q are zero-filled in A (TMA OOB), so they add 0.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <stdlib.h>

#include <algorithm>

#include "gemm_common.cuh"
#include "gemm_engines.cuh"
#include "tc_ptx.cuh"

namespace bf {
namespace wgt {

using namespace tcu;

constexpr int BK = 32;
#ifndef WGT_SACC
#define WGT_SACC 1
#endif
// with the separate small-term accumulator the accumulator takes 2*NP TMEM
// columns and three A stages fit; without it NP columns and four
constexpr int kStages = WGT_SACC ? 3 : 4;     // B (smem) and A (TMEM) stages, per k-block
constexpr int kRawStages = WGT_SACC ? 6 : 4;  // raw dY tiles (smem), TMA'd ahead of the MMA
// warps: 0 TMA, 1 MMA (+ TMEM allocation), 4-5 split (TMEM lane quarters 0-1 =
// kout rows 0-63), 2-3 and 6-13 producers (10), 14-17 epilogue (all four lane
// quarters)
constexpr int kTmaWarp = 0, kMmaWarp = 1, kSplitWarp0 = 4, kSplitWarps = 2, kProdWarp0 = 6;
constexpr int kProdWarps = 8, kEpiWarp0 = kProdWarp0 + kProdWarps, kEpiWarps = 4;
constexpr int kThreads = (kEpiWarp0 + kEpiWarps) * 32;
constexpr int kProducers = (kProdWarps + 2) * 32;
__device__ __forceinline__ bool is_producer(int warp) {
  return warp == 2 || warp == 3 || (warp >= kProdWarp0 && warp < kProdWarp0 + kProdWarps);
}
constexpr int kRawBytes = 64 * 128;  // raw dY tile: <= 64 kout rows x 32 floats
constexpr int kWinSlots = 4;         // window staging ring: cp.async kWinSlots-1 k-blocks ahead

struct Geo {
  int N, C, H, W, K, R, S, P, Q, st, pad;
  int CR, CRS, NP;      // (c, r) windows, rows (c, r, s), rows padded to 16
  int nq, nkb;          // k-blocks per output row, total k-blocks
  int nch;              // 16-byte chunks per window
  int kbps, splits;     // k-blocks per unit, units
  int stage_bytes;      // B stage: [B big | B small]
  int win_floats;       // staging floats per window (4 * nch)
  int abase;            // first TMEM column of the A ring (after the 2*NP accumulator columns)
};

__device__ __forceinline__ float lds_f32(uint32_t a) {
  float v;
  asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ float4 lds_v4(uint32_t a) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "r"(a));
  return v;
}
__device__ __forceinline__ void sts_v4(uint32_t a, float4 v) {
  asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(a), "f"(v.x), "f"(v.y), "f"(v.z),
               "f"(v.w)
               : "memory");
}
__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src, bool ok) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src),
               "r"(ok ? 16 : 0)
               : "memory");
}

__global__ void __launch_bounds__(kThreads, 1)
    wgt_kernel(const __grid_constant__ CUtensorMap dymap, const float* __restrict__ x, Geo g,
               EpiPartial part, float* __restrict__ bias_part) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint8_t* rawbuf = base + kStages * g.stage_bytes;                        // kRawStages tiles
  float* staging = reinterpret_cast<float*>(rawbuf + kRawStages * kRawBytes);
  uint64_t* bars = reinterpret_cast<uint64_t*>(staging + kWinSlots * g.CR * g.win_floats);
  uint64_t* raw_full = bars;                     // TMA landed the raw dY tile
  uint64_t* raw_free = raw_full + kRawStages;    // split warps read it
  uint64_t* a_full = raw_free + kRawStages;      // split warps wrote A big / small to TMEM
  uint64_t* b_full = a_full + kStages;           // producers wrote B big / small
  uint64_t* empty = b_full + kStages;            // MMAs of the stage done
  uint64_t* acc_full = empty + kStages;
  uint64_t* acc_empty = acc_full + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 1);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int NP = g.NP;

  if (warp == kMmaWarp) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
        smem_u32(tmem_slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (threadIdx.x == 0) {
    for (int s = 0; s < kRawStages; ++s) {
      mbar_init(&raw_full[s], 1);
      mbar_init(&raw_free[s], kSplitWarps * 32);
    }
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&a_full[s], kSplitWarps * 32);
      mbar_init(&b_full[s], kProducers);
      mbar_init(&empty[s], 1);
    }
    mbar_init(acc_full, 1);
    mbar_init(acc_empty, kEpiWarps * 32);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&dymap)) : "memory");
  }
  // zero the B stages once: rows >= CRS are never written again
  for (int i = threadIdx.x; i < kStages * g.stage_bytes / 16; i += kThreads)
    reinterpret_cast<float4*>(base)[i] = make_float4(0.f, 0.f, 0.f, 0.f);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  // TMEM lanes 64-127 of the A ring (kout rows 64..127 of the M = 128 tile) stay
  // zero: written once by the warps of lane quarters 2 and 3
  if (warp == kProdWarp0 || warp == kProdWarp0 + 1) {  // quarters 2, 3
    float z[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) z[j] = 0.f;
    const uint32_t la = tmem + ((uint32_t)((warp & 3) * 32) << 16);
    for (int col = g.abase; col < g.abase + kStages * 64; col += 16) tmem_st16(la + col, z);
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();

  auto kb_coords = [&](int kb, int& img, int& p, int& q0) {
    const int per_img = g.P * g.nq;
    img = kb / per_img;
    const int rem = kb - img * per_img;
    p = rem / g.nq;
    q0 = (rem - p * g.nq) * BK;
  };

  if (warp == kTmaWarp) {
    // ======================= raw dY tiles by TMA =======================
    if (lane == 0) {
      int s = 0;
      uint32_t ph = 0;
      for (int u = blockIdx.x; u < g.splits; u += gridDim.x) {
        const int kb0 = u * g.kbps, nk = min(g.kbps, g.nkb - kb0);
        int img, p, q0;
        kb_coords(kb0, img, p, q0);  // then advanced incrementally
        for (int i = 0; i < nk; ++i) {
          mbar_wait(&raw_free[s], ph ^ 1);
          mbar_arrive_expect_tx(&raw_full[s], (uint32_t)(g.K * 128));
          if (i > 0 && (q0 += BK) == g.nq * BK) {
            q0 = 0;
            if (++p == g.P) {
              p = 0;
              ++img;
            }
          }
          asm volatile(
              "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes"
              " [%0], [%1, {%2, %3, %4, %5}], [%6];" ::"r"(smem_u32(rawbuf + s * kRawBytes)),
              "l"(reinterpret_cast<uint64_t>(&dymap)), "r"(q0), "r"(p), "r"(0), "r"(img),
              "r"(smem_u32(&raw_full[s]))
              : "memory");
          if (++s == kRawStages) {
            s = 0;
            ph ^= 1;
          }
        }
      }
    }
    __syncwarp();
  } else if (warp >= kSplitWarp0 && warp < kSplitWarp0 + kSplitWarps) {
    // ======================= A: dY row -> TMEM big / small, bias sums =======================
    // thread = kout row m = TMEM lane (quarters 0, 1)
    const int m = (warp & 3) * 32 + lane;
    const bool live = m < g.K;
    const uint32_t raw_a = smem_u32(rawbuf);
    const uint32_t la = tmem + ((uint32_t)((warp & 3) * 32) << 16);
    int rs = 0, s = 0;
    uint32_t rph = 0, ph = 0;
    for (int u = blockIdx.x; u < g.splits; u += gridDim.x) {
      const int kb0 = u * g.kbps, nk = min(g.kbps, g.nkb - kb0);
      float bsum = 0.f;
      for (int i = 0; i < nk; ++i) {
        mbar_wait(&raw_full[rs], rph);
        float big[32], small[32];
        const uint32_t row = raw_a + (uint32_t)(rs * kRawBytes + m * 128);
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
          if (live) v = lds_v4(row + (uint32_t)((c ^ (m & 7)) << 4));
          big[4 * c + 0] = v.x; big[4 * c + 1] = v.y; big[4 * c + 2] = v.z; big[4 * c + 3] = v.w;
          const float4 r = tf32_small4(v);
          small[4 * c + 0] = r.x; small[4 * c + 1] = r.y; small[4 * c + 2] = r.z;
          small[4 * c + 3] = r.w;
          bsum = __fadd_rn(bsum, __fadd_rn(__fadd_rn(v.x, v.y), __fadd_rn(v.z, v.w)));
        }
        mbar_arrive(&raw_free[rs]);
        if (++rs == kRawStages) {
          rs = 0;
          rph ^= 1;
        }
        mbar_wait(&empty[s], ph ^ 1);
        tc_fence_after();
        const uint32_t acol = g.abase + s * 64;
        tmem_st16(la + acol, *reinterpret_cast<const float(*)[16]>(&big[0]));
        tmem_st16(la + acol + 16, *reinterpret_cast<const float(*)[16]>(&big[16]));
        tmem_st16(la + acol + 32, *reinterpret_cast<const float(*)[16]>(&small[0]));
        tmem_st16(la + acol + 48, *reinterpret_cast<const float(*)[16]>(&small[16]));
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        tc_fence_before();
        mbar_arrive(&a_full[s]);
        if (++s == kStages) {
          s = 0;
          ph ^= 1;
        }
      }
      if (bias_part && live) bias_part[(size_t)m * g.splits + u] = bsum;
    }
  } else if (warp == kMmaWarp) {
    // ======================= MMA issuer =======================
    const uint32_t idesc = tf32_idesc(NP);
    int s = 0, local = 0;
    uint32_t ph = 0;
    for (int u = blockIdx.x; u < g.splits; u += gridDim.x, ++local) {
      const int kb0 = u * g.kbps, nk = min(g.kbps, g.nkb - kb0);
      mbar_wait(acc_empty, (local & 1) ^ 1);
      tc_fence_after();
      const uint32_t dbig = tmem, dsm = tmem + (uint32_t)NP;
      for (int i = 0; i < nk; ++i) {
        mbar_wait(&a_full[s], ph);
        mbar_wait(&b_full[s], ph);
        tc_fence_after();
        const uint32_t st = smem_u32(base + s * g.stage_bytes);
        const uint64_t bb = sw128_desc(st), bs = sw128_desc(st + NP * 128);
        const uint32_t ab = tmem + (uint32_t)(g.abase + s * 64), as = ab + 32;
        if (elect_one()) {
          if (WGT_SACC) {
            if (i == 0) {
              mma_ts_flag<0>(dbig, ab, bb, idesc);
              mma_ts_flag<0>(dsm, ab, bs, idesc);
            } else {
              mma_ts_flag<1>(dbig, ab, bb, idesc);
              mma_ts_flag<1>(dsm, ab, bs, idesc);
            }
            mma_ts_flag<1>(dsm, as, bb, idesc);
#pragma unroll
            for (int ks = 1; ks < BK / 8; ++ks) {
              const uint64_t k2 = (uint64_t)((ks * 32) >> 4);
              mma_ts_flag<1>(dbig, ab + ks * 8, bb + k2, idesc);
              mma_ts_flag<1>(dsm, ab + ks * 8, bs + k2, idesc);
              mma_ts_flag<1>(dsm, as + ks * 8, bb + k2, idesc);
            }
          } else {  // all three products into one accumulator (small terms first)
            if (i == 0)
              mma_ts_flag<0>(dbig, as, bb, idesc);
            else
              mma_ts_flag<1>(dbig, as, bb, idesc);
            mma_ts_flag<1>(dbig, ab, bs, idesc);
            mma_ts_flag<1>(dbig, ab, bb, idesc);
#pragma unroll
            for (int ks = 1; ks < BK / 8; ++ks) {
              const uint64_t k2 = (uint64_t)((ks * 32) >> 4);
              mma_ts_flag<1>(dbig, as + ks * 8, bb + k2, idesc);
              mma_ts_flag<1>(dbig, ab + ks * 8, bs + k2, idesc);
              mma_ts_flag<1>(dbig, ab + ks * 8, bb + k2, idesc);
            }
          }
          tc_commit(&empty[s]);
        }
        __syncwarp();
        if (++s == kStages) {
          s = 0;
          ph ^= 1;
        }
      }
      if (elect_one()) tc_commit(acc_full);
      __syncwarp();
    }
  } else if (is_producer(warp)) {
    // ======================= B: the im2col of x =======================
    const int t = (warp < kProdWarp0 ? warp - 2 : warp - kProdWarp0 + 2) * 32 + lane;
    const uint32_t stg0 = smem_u32(staging), base_a = smem_u32(base);
    const int wf = g.win_floats;
    // this thread's window chunks (fixed for every k-block): ids t, t + 256, ...
    // of the CR x nch chunks -> (c, r, f); only the k-block's (img, p, q0) vary
    constexpr int kMaxIds = 4;
    // per chunk: its row r and column 4f (bounds), its offset from the
    // k-block's window origin x[img][0][st*p - pad][a0] and its staging slot
    int id_r[kMaxIds], id_f4[kMaxIds], id_off[kMaxIds], id_dst[kMaxIds], nid = 0;
    for (int id = t; id < g.CR * g.nch && nid < kMaxIds; id += kProducers, ++nid) {
      const int cr = id / g.nch, f = id - cr * g.nch, c = cr / g.R;
      id_r[nid] = cr - c * g.R;
      id_f4[nid] = 4 * f;
      id_off[nid] = (c * g.H + id_r[nid]) * g.W + 4 * f;
      id_dst[nid] = (cr * wf + 4 * f) * 4;
    }
    // k-block cursors over this CTA's sequence (unit u's kb0 .. kb0+nk-1, then
    // unit u + gridDim.x's): (img, p, q-block) advance incrementally -- the
    // per-k-block divisions cost the producers ~100 instructions per k-block
    struct Cur {
      int u, i, nk, img, p, qb;
    };
    auto cur_init = [&](Cur& c, int u) {
      c.u = u;
      c.i = 0;
      if (u < g.splits) {
        const int kb0 = u * g.kbps;
        c.nk = min(g.kbps, g.nkb - kb0);
        int q0;
        kb_coords(kb0, c.img, c.p, q0);
        c.qb = q0 / BK;
      }
    };
    auto cur_next = [&](Cur& c) {
      if (++c.i >= c.nk) {
        cur_init(c, c.u + gridDim.x);
      } else if (++c.qb == g.nq) {
        c.qb = 0;
        if (++c.p == g.P) {
          c.p = 0;
          ++c.img;
        }
      }
    };
    // stage the (c, r) windows of the cursor's k-block into staging slot `slot`
    auto issue = [&](const Cur& c, int slot) {
      if (c.u < g.splits) {
        const int a0 = (g.st * c.qb * BK - g.pad) & ~3;  // 16-byte aligned window start
        const uint32_t sbase = stg0 + (uint32_t)(slot * g.CR * wf * 4);
        const int ih0 = g.st * c.p - g.pad;
        const float* xo = x + ((int64_t)c.img * g.C * g.H + ih0) * g.W + a0;
#pragma unroll
        for (int j = 0; j < kMaxIds; ++j) {
          if (j < nid) {
            const bool ok = (unsigned)(ih0 + id_r[j]) < (unsigned)g.H &&
                            (unsigned)(a0 + id_f4[j]) < (unsigned)g.W;
            cp_async16(sbase + (uint32_t)id_dst[j], ok ? xo + id_off[j] : x, ok);
          }
        }
      }
      asm volatile("cp.async.commit_group;" ::: "memory");
    };
    Cur ic;  // the issue cursor runs kWinSlots-1 k-blocks ahead of use
    cur_init(ic, blockIdx.x);
#pragma unroll 1
    for (int d = 0; d < kWinSlots - 1; ++d) {
      issue(ic, d);
      if (ic.u < g.splits) cur_next(ic);
    }
    // B-image work: thread t writes 16-byte chunk c = t & 7 (pixels 4c..4c+3) of
    // rows n = (t >> 3) + 32 j, n = cr*S + s -- the window offsets and
    // swizzled destinations are fixed for every k-block, so precomputed
    constexpr int kMaxRows = 8;  // CRS <= 256 rows, 32 row groups
    int row_win[kMaxRows] = {}, row_dst[kMaxRows] = {}, nrow = 0;
    {
      const int c = t & 7;
      for (int n = t >> 3; n < g.CRS && nrow < kMaxRows; n += kProducers / 8, ++nrow) {
        const int cr = n / g.S, ss = n - cr * g.S;
        row_win[nrow] = (cr * wf + ss + g.st * 4 * c) * 4;  // bytes
        row_dst[nrow] = (int)sw_off(n, c);
      }
    }
    int s = 0, slot = 0;
    uint32_t ph = 0;
    Cur mc;
    cur_init(mc, blockIdx.x);
    while (mc.u < g.splits) {
      {
        // this k-block's windows are the oldest of kWinSlots-1 groups in flight;
        // the barrier also retires every thread's reads of the previous k-block,
        // whose slot the next issue refills
        asm volatile("cp.async.wait_group %0;" ::"n"(kWinSlots - 2) : "memory");
        named_sync(1, kProducers);
        issue(ic, (slot + kWinSlots - 1) % kWinSlots);
        if (ic.u < g.splits) cur_next(ic);
        const int q0 = mc.qb * BK;
        const int o = (g.st * q0 - g.pad) - ((g.st * q0 - g.pad) & ~3);
        cur_next(mc);
        mbar_wait(&empty[s], ph ^ 1);
        // shared-space 32-bit addressing (generic pointers cost 64-bit address
        // arithmetic and generic loads / stores per element)
        const uint32_t bbig = base_a + (uint32_t)(s * g.stage_bytes), bsml = bbig + NP * 128;
        const uint32_t win_a = stg0 + (uint32_t)((slot * g.CR * wf + o) * 4);
        const uint32_t st4 = (uint32_t)g.st * 4;
#pragma unroll
        for (int j = 0; j < kMaxRows; ++j) {
          if (j < nrow) {
            const uint32_t a = win_a + (uint32_t)row_win[j];
            const float4 v = make_float4(lds_f32(a), lds_f32(a + st4), lds_f32(a + 2 * st4),
                                         lds_f32(a + 3 * st4));
            sts_v4(bbig + (uint32_t)row_dst[j], v);
            sts_v4(bsml + (uint32_t)row_dst[j], tf32_small4(v));
          }
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        mbar_arrive(&b_full[s]);
        if (++slot == kWinSlots) slot = 0;
        if (++s == kStages) {
          s = 0;
          ph ^= 1;
        }
      }
    }
    asm volatile("cp.async.wait_all;" ::: "memory");
  } else if (warp >= kEpiWarp0) {
    // ======================= epilogue =======================
    const int q = warp & 3;
    int local = 0;
    for (int u = blockIdx.x; u < g.splits; u += gridDim.x, ++local) {
      mbar_wait(acc_full, local & 1);
      tc_fence_after();
      const int m = q * 32 + lane;
      const bool live = m < g.K;
      const uint32_t taddr = tmem + ((uint32_t)(q * 32) << 16);
      const RowPtr rp = live ? part.row(u, m) : RowPtr{nullptr, 0.f};
#pragma unroll 1
      for (int c0 = 0; c0 < NP; c0 += 16) {
        uint32_t v[16], sv[16];
        tmem_ld16(taddr + (uint32_t)c0, v);
        if (WGT_SACC) {
          tmem_ld16(taddr + (uint32_t)(NP + c0), sv);
#pragma unroll
          for (int j = 0; j < 16; ++j)
            v[j] = __float_as_uint(__fadd_rn(__uint_as_float(v[j]), __uint_as_float(sv[j])));
        }
        if (live) part.store16(rp, c0, v, g.CRS - c0);
      }
      tc_fence_before();
      mbar_arrive(acc_empty);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == kMmaWarp) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
  }
}

// dW[m][n] = v (m = kout, n = (c, r, s)): the reduction's final epilogue
struct EpiRowMajor {
  float* out;
  int ld;
  __device__ __forceinline__ void operator()(int m, int n, float v) const {
    out[(int64_t)m * ld + n] = v;
  }
};

static bool make_dy4_map(CUtensorMap* map, const float* dy, int N, int K, int P, int Q) {
  auto fn = tma_encode_fn();
  if (!fn) return false;
  cuuint64_t dims[4] = {(cuuint64_t)Q, (cuuint64_t)P, (cuuint64_t)K, (cuuint64_t)N};
  cuuint64_t strides[3] = {(cuuint64_t)Q * 4, (cuuint64_t)P * Q * 4, (cuuint64_t)K * P * Q * 4};
  cuuint32_t box[4] = {32, 1, (cuuint32_t)K, 1};
  cuuint32_t estr[4] = {1, 1, 1, 1};
  return fn(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, const_cast<float*>(dy), dims, strides, box,
            estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

}  // namespace wgt

bool wgrad_t_enabled() {
  const char* e = getenv("PURINE_B200_WGRAD_T");
  return !(e && *e && atoi(e) == 0);
}

// -1 when the shape is not taken
int wgrad_t_conv(const ConvShape& g, const float* x, const float* dy, float* dw, float* db,
                 bool* db_done, float* ws, int64_t ws_bytes, cudaStream_t st, const char* what) {
  using namespace wgt;
  if (db_done) *db_done = false;
  if (!wgrad_t_enabled()) return -1;
  const int CRS = g.C * g.R * g.S;
  if (g.K > 64 || g.K < 8 || CRS > 256 || g.S > 8 || g.W % 4 || g.Q % 4 ||
      ((reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(dy)) & 15))
    return -1;
  Geo q{};
  q.N = g.N; q.C = g.C; q.H = g.H; q.W = g.W; q.K = g.K; q.R = g.R; q.S = g.S;
  q.P = g.P; q.Q = g.Q; q.st = g.stride; q.pad = g.pad;
  q.CR = g.C * g.R;
  q.CRS = CRS;
  q.NP = (CRS + 15) / 16 * 16;
  q.nq = (g.Q + BK - 1) / BK;
  q.nkb = g.N * g.P * q.nq;
  q.nch = (3 + g.stride * (BK - 1) + g.S + 3) / 4;
  q.win_floats = q.nch * 4;
  q.stage_bytes = 2 * q.NP * 128;
  q.abase = ((WGT_SACC ? 2 : 1) * q.NP + 63) / 64 * 64;
  if (g.K > 64 || q.abase + kStages * 64 > 512 || q.CR * q.nch > 4 * kProducers) return -1;
  const int smem_cap = 227 * 1024;
  const int smem = 1024 + kStages * q.stage_bytes + kRawStages * kRawBytes +
                   kWinSlots * q.CR * q.win_floats * 4 + (2 * kRawStages + 3 * kStages + 2) * 8 +
                   64;
  if (smem > smem_cap) return -1;
  // units: chains of at most max_chain_kb() k-blocks, balanced over the grid
  const int sms = gemm_sm_budget();
  const int64_t chain = std::max<int64_t>(1, chain_min_splits(q.nkb, WGT_SACC != 0));
  const int64_t bias_bytes = db ? ((int64_t)g.K * kMaxSplits * 4 + 1023) / 1024 * 1024 : 0;
  if (!ws || ws_bytes < bias_bytes) return -1;
  const int64_t by_ws = (ws_bytes - bias_bytes) / ((int64_t)g.K * CRS * 4);
  const int64_t cap = std::min<int64_t>(by_ws, kMaxSplits);
  int64_t splits = std::max<int64_t>(chain, std::min<int64_t>(sms, q.nkb));
  splits = std::min(splits, cap);
  splits = balance_splits(1, q.nkb, splits, cap, sms);
  if (splits < 1) return -1;
  q.kbps = (int)((q.nkb + splits - 1) / splits);
  q.splits = (q.nkb + q.kbps - 1) / q.kbps;
  CUtensorMap dymap;
  if (!make_dy4_map(&dymap, dy, g.N, g.K, g.P, g.Q)) return -1;
  float* bias_ws = db ? ws : nullptr;
  float* part_ws = reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(ws) + bias_bytes);
  static bool configured = false;
  if (!configured) {
    BF_CUDA(cudaFuncSetAttribute(wgt_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 smem_cap),
            "wgrad-T smem attribute");
    configured = true;
  }
  EpiPartial part{part_ws, g.K, CRS};
  const int grid = std::min(q.splits, sms);
  wgt_kernel<<<grid, kThreads, smem, st>>>(dymap, x, q, part, bias_ws);
  if (int rc = check_launch(what)) return rc;
  splitk_reduce<EpiRowMajor>(part_ws, q.splits, g.K, CRS, EpiRowMajor{dw, CRS}, st);
  if (int rc = check_launch(what)) return rc;
  if (db) {
    tcu::bias_blocks_finish_kernel<<<g.K, 256, 0, st>>>(bias_ws, q.splits, db);
    if (int rc = check_launch(what)) return rc;
    if (db_done) *db_done = true;
  }
  return 0;
}

}  // namespace bf
