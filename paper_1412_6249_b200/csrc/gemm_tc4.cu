// tcgen05 engine v4: TMA-fed 1x1 convolutions (forward and data gradient), 3xTF32.
//
// A 1x1 stride-1 convolution is, per image, a plain GEMM on the NCHW tensors:
//   fwd   y[n][k][p] = sum_c w[k][c] x[n][c][p]      (ops.py:281-297)
//   dgrad dx[n][c][p] = sum_k w[k][c] dy[n][k][p]    (ops.py:332-343)
// With the output pixel as the MMA M index, the activation operand is
// "MN-major" in memory (pixels contiguous, channels strided) -- a layout the
// tensor core reads directly for kind::tf32 (instruction descriptor bit 15;
// shared-memory layout "128B swizzle, 32B atoms", see mn_sw128_32b_desc).
// So nothing is gathered: a TMA warp streams 128-pixel x 32-channel boxes
// straight from x (or dy) into 128B-swizzled shared memory, and the weights
// come pre-packed (tc_ptx.cuh pack_b_kernel) by bulk copy, as in engine v2.
//
// 3xTF32 split of the activation: the tensor core ignores the 13 low mantissa
// bits of a kind::tf32 operand, so the raw TMA tile IS the "big" operand;
// four "split" warps only compute small = x - trunc(x) (exact) into a second
// tile: one 16-byte load, four AND + four FADD and one 16-byte store per four
// elements.  MMAs per k-step of 8: small*big + big*small + big*big, both
// operands from shared memory.
//
// Warp roles (14 warps, 4 per SM sub-partition -> up to 128 registers):
//   warp 0        TMA / bulk-copy issuer (one thread)
//   warps 1-4     split warps
//   warp 5        MMA issuer (one thread) + TMEM allocator
//   warps 6-13    epilogue: TMEM -> registers -> NCHW global stores (fused
//                 bias / ReLU exactly as engine v2's EpiNCHW)
// Tiles never straddle images (the TMA box is per image; pixels past the
// image end are zero-filled and their rows discarded).
#include <cuda.h>
#include <cudaTypedefs.h>

#include <stdlib.h>

#include <algorithm>

#include "gemm_common.cuh"
#include "gemm_engines.cuh"
#include "tc_ptx.cuh"

namespace bf {

static bool tc4_sacc_enabled() {
  const char* e = getenv("PURINE_B200_SACC");
  return !(e && *e && atoi(e) == 0);
}

namespace tc4 {

using namespace tcu;

constexpr int BK = 32;
constexpr int kMaxStages = 6;
constexpr int kTmaWarp = 0, kSplitWarp0 = 1, kSplitWarps = 4, kMmaWarp = 5, kEpiWarp0 = 6;
constexpr int kEpiWarps = 8;
constexpr int kThreads = (kEpiWarp0 + kEpiWarps) * 32;
constexpr int kABytes = BM * BK * 4;  // one raw activation tile (16 KB)

struct Work {
  int PQ, tiles_img, N_img, Nout, K, BN, ntiles, nkb, kbps, splits, units, nst, nacc;
  int stage_bytes, b_bytes;
  int tmem_cols;  // 512, or 256 when two CTAs share an SM (two MMA issuers)
  int sacc;       // 1: separate small-term accumulator (see the MMA issuer)
  int accw;       // TMEM columns per accumulator buffer (BN, or 2*BN with sacc)
  // K segments (grouped data gradient): k-block kb < seg_kb[s + 1] of segment s
  // comes from activation map s at k-block kb - seg_kb[s] (zero-filled rows past
  // that tensor's channel count)
  int nseg;
  int seg_kb[kMaxSeg + 1];
};

struct ActMaps {
  CUtensorMap m[kMaxSeg];
};

// MN-major tf32 operand: the only smem layout the tensor core accepts is
// "128B swizzle with 32B atomicity" (descriptor layout type 1; TMA
// CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B writes it): 128-byte K rows of 32
// MN-elements whose 32-byte granules are permuted by row, 4-row (512 B) atoms.
// 32-element MN chunks (one TMA box each) 4 KB apart = LBO; 4-row K groups
// 512 B apart = SBO.  Verified bit-exactly by tools/mn_probe.cu.
__device__ __forceinline__ uint64_t mn_sw128_32b_desc(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)(4096 >> 4) << 16;
  d |= (uint64_t)(512 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)1 << 61;
  return d;
}

template <int ACC>
__device__ __forceinline__ void mma_ss(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc) {
  asm volatile("tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, %4;" ::"r"(d), "l"(a),
               "l"(b), "r"(idesc), "n"(ACC)
               : "memory");
}

__device__ __forceinline__ void unit_coords(const Work& w, int u, int& img, int& pt, int& nt,
                                            int& sp) {
  // divisions by 1 (no split-K, one channel tile, one pixel tile) skipped:
  // warp-uniform branches, ~20 instructions saved per division per unit
  auto dm = [](int x, int d, int& q, int& r) {
    if (d == 1) {
      q = x;
      r = 0;
    } else {
      q = x / d;
      r = x - q * d;
    }
  };
  int r, r2;
  dm(u, w.splits, r, sp);
  dm(r, w.ntiles, r2, nt);
  dm(r2, w.tiles_img, img, pt);
}

template <class Epi>
__global__ void __launch_bounds__(kThreads, 2)
    tc4_kernel(const __grid_constant__ ActMaps amaps, Work w, const uint8_t* __restrict__ bpack,
               Epi epi, EpiPartial part) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  const int BN = w.BN;
  // stage s: [A raw | A small | B big | B small]
  uint64_t* raw_full = reinterpret_cast<uint64_t*>(base + w.nst * w.stage_bytes);
  uint64_t* split_full = raw_full + kMaxStages;
  uint64_t* empty = split_full + kMaxStages;
  uint64_t* acc_full = empty + kMaxStages;
  uint64_t* acc_empty = acc_full + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 2);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (warp == kMmaWarp) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
        smem_u32(tmem_slot)), "r"(w.tmem_cols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (threadIdx.x == 0) {
    for (int s = 0; s < kMaxStages; ++s) {
      mbar_init(&raw_full[s], 1);
      mbar_init(&split_full[s], kSplitWarps * 32);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&acc_full[b], 1);
      mbar_init(&acc_empty[b], kEpiWarps * 32);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    for (int i = 0; i < w.nseg; ++i)
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&amaps.m[i]))
                   : "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == kTmaWarp) {
    // ======================= TMA issue =======================
    if (lane == 0) {
      int rs = 0;
      uint32_t rph = 0;
      for (int u = blockIdx.x; u < w.units; u += gridDim.x) {
        int img, pt, nt, sp;
        unit_coords(w, u, img, pt, nt, sp);
        const int kb0 = sp * w.kbps, nk = min(w.kbps, w.nkb - kb0);
        for (int i = 0; i < nk; ++i) {
          const int s = rs;
          const uint32_t sph = rph;
          if (++rs == w.nst) {
            rs = 0;
            rph ^= 1;
          }
          mbar_wait(&empty[s], sph ^ 1);
          mbar_arrive_expect_tx(&raw_full[s], (uint32_t)(kABytes + w.b_bytes));
          uint8_t* st = base + s * w.stage_bytes;
          const int kb = kb0 + i;
          int sg = 0;
#pragma unroll
          for (int q = 1; q < kMaxSeg; ++q) sg += (q < w.nseg && kb >= w.seg_kb[q]) ? 1 : 0;
          const CUtensorMap* am = &amaps.m[sg];
          const int kc = (kb - w.seg_kb[sg]) * BK;
#pragma unroll
          for (int j = 0; j < BM / 32; ++j)
            tma_load_3d(smem_u32(st + j * 4096), am, pt * BM + j * 32, kc, img, &raw_full[s]);
          bulk_g2s(smem_u32(st + 2 * kABytes),
                   bpack + ((size_t)nt * w.nkb + kb0 + i) * w.b_bytes, (uint32_t)w.b_bytes,
                   &raw_full[s]);
        }
      }
    }
    __syncwarp();
  } else if (warp >= kSplitWarp0 && warp < kSplitWarp0 + kSplitWarps) {
    // ======================= split: small = x - trunc(x) =======================
    const int t = threadIdx.x - kSplitWarp0 * 32;
    int rs = 0;
    uint32_t rph = 0;
    for (int u = blockIdx.x; u < w.units; u += gridDim.x) {
      int img, pt, nt, sp;
      unit_coords(w, u, img, pt, nt, sp);
      const int nk = min(w.kbps, w.nkb - sp * w.kbps);
      for (int i = 0; i < nk; ++i) {
        const int s = rs;
        const uint32_t sph = rph;
        if (++rs == w.nst) {
          rs = 0;
          rph ^= 1;
        }
        mbar_wait(&raw_full[s], sph);
        const float4* src = reinterpret_cast<const float4*>(base + s * w.stage_bytes);
        float4* dst = reinterpret_cast<float4*>(base + s * w.stage_bytes + kABytes);
#pragma unroll
        for (int q = 0; q < kABytes / 16 / (kSplitWarps * 32); ++q) {
          const float4 v = src[q * kSplitWarps * 32 + t];
          const float4 r = tf32_small4(v);
          dst[q * kSplitWarps * 32 + t] = r;
        }
        // generic-proxy smem writes -> visible to the tensor core (async proxy)
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        mbar_arrive(&split_full[s]);
      }
    }
  } else if (warp == kMmaWarp) {
    // ======================= MMA issue =======================
    // whole warp walks the schedule; one elected lane issues (see gemm_tc2.cu)
    {
      // A MN-major (bit 15), B K-major; M = 128, N = BN
      const uint32_t idesc = tf32_idesc(BN) | (1u << 15);
      // sacc: the B stage holds [B big rows | B small rows] contiguously, so ONE
      // N = 2*BN instruction computes A_big*B_big into columns [0, BN) and
      // A_big*B_small into [BN, 2BN); A_small*B_big accumulates into [BN, 2BN)
      // too.  Two instructions per k-step instead of three (the narrow tiles
      // are issue-bound), and the big accumulator takes one round-toward-zero
      // accumulation per k-step instead of three (the small terms' own
      // truncation is 2^-11 smaller); the epilogue adds the halves in fp32 RN.
      const uint32_t idesc2 = tf32_idesc(2 * BN) | (1u << 15);
      int rs = 0, local = 0;
      uint32_t rph = 0;
      for (int u = blockIdx.x; u < w.units; u += gridDim.x, ++local) {
        int img, pt, nt, sp;
        unit_coords(w, u, img, pt, nt, sp);
        const int nk = min(w.kbps, w.nkb - sp * w.kbps);
        const int b = local % w.nacc;
        const uint32_t use = local / w.nacc;
        mbar_wait(&acc_empty[b], (use & 1) ^ 1);
        tc_fence_after();
        const uint32_t dacc = tmem + (uint32_t)(b * w.accw);
        for (int i = 0; i < nk; ++i) {
          const int s = rs;
          const uint32_t sph = rph;
          if (++rs == w.nst) {
            rs = 0;
            rph ^= 1;
          }
          mbar_wait(&split_full[s], sph);
          tc_fence_after();
          const uint32_t st = smem_u32(base + s * w.stage_bytes);
          const uint64_t abig = mn_sw128_32b_desc(st), asmall = mn_sw128_32b_desc(st + kABytes);
          const uint64_t bbig = sw128_desc(st + 2 * kABytes);
          const uint64_t bsmall = sw128_desc(st + 2 * kABytes + BN * 128);
          if (elect_one()) {
            // k-step ks (8 K rows): A start + 1 KB (two 4-row atoms), B start + 32 B
            if (w.sacc) {
              const uint32_t dsm = dacc + (uint32_t)BN;
              if (i == 0)
                mma_ss<0>(dacc, abig, bbig, idesc2);
              else
                mma_ss<1>(dacc, abig, bbig, idesc2);
              mma_ss<1>(dsm, asmall, bbig, idesc);
#pragma unroll
              for (int ks = 1; ks < BK / 8; ++ks) {
                const uint64_t ak = (uint64_t)((ks * 1024) >> 4), bk = (uint64_t)((ks * 32) >> 4);
                mma_ss<1>(dacc, abig + ak, bbig + bk, idesc2);
                mma_ss<1>(dsm, asmall + ak, bbig + bk, idesc);
              }
            } else {
              if (i == 0)
                mma_ss<0>(dacc, asmall, bbig, idesc);
              else
                mma_ss<1>(dacc, asmall, bbig, idesc);
              mma_ss<1>(dacc, abig, bsmall, idesc);
              mma_ss<1>(dacc, abig, bbig, idesc);
#pragma unroll
              for (int ks = 1; ks < BK / 8; ++ks) {
                const uint64_t ak = (uint64_t)((ks * 1024) >> 4), bk = (uint64_t)((ks * 32) >> 4);
                mma_ss<1>(dacc, asmall + ak, bbig + bk, idesc);
                mma_ss<1>(dacc, abig + ak, bsmall + bk, idesc);
                mma_ss<1>(dacc, abig + ak, bbig + bk, idesc);
              }
            }
            tc_commit(&empty[s]);
          }
          __syncwarp();
        }
        if (elect_one()) tc_commit(&acc_full[b]);
        __syncwarp();
      }
    }
  } else {
    // ======================= epilogue =======================
    const int ew = warp - kEpiWarp0;
    const int q = warp & 3;
    const int half = ew >> 2;
    int local = 0;
    for (int u = blockIdx.x; u < w.units; u += gridDim.x, ++local) {
      int img, pt, nt, sp;
      unit_coords(w, u, img, pt, nt, sp);
      const int b = local % w.nacc;
      const uint32_t use = local / w.nacc;
      mbar_wait(&acc_full[b], use & 1);
      tc_fence_after();
      const int pix = pt * BM + q * 32 + lane;
      const bool live = pix < w.PQ;
      const int m = img * w.PQ + pix;
      const int n0 = nt * BN;
      const int cols = BN / 2;
      const uint32_t taddr = tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(b * w.accw);
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
          const int nlim = w.Nout - (n0 + c0);
          if (w.splits > 1) {
            part.store16(rp, n0 + c0, v, nlim);
          } else {
            epi.store16(rp, n0 + c0, v, nlim);
          }
        }
      }
      tc_fence_before();
      mbar_arrive(&acc_empty[b]);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == kMmaWarp) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                 "r"(w.tmem_cols));
  }
}

// [imgs][rows][PQ] fp32 activation, box {32 pixels, 32 rows, 1}, 128B swizzle with
// 32B atomicity (the MN-major tf32 layout, see mn_sw128_32b_desc)
static bool make_act_map(CUtensorMap* map, const float* p, int PQ, int rows, int imgs) {
  return make_nchw_map(map, p, PQ, rows, imgs, BK, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B);
}

inline int pick_bn(int N, int& ntiles) {
  ntiles = (N + 255) / 256;
  int per = (N + ntiles - 1) / ntiles;
  return (per + 31) / 32 * 32;
}

// act: [imgs][K][PQ]; B(n, k) via lbp (pre-packed); D[m = img*PQ + pix][n] -> epi
// act[s]: [imgs][kseg[s]][PQ], K = sum of kseg rounded up to 32 per segment
template <class LBP, class Epi>
int launch_seg(int nseg, const float* const* act, const int* kseg, int imgs, int PQ, int Nout,
               const LBP& lbp, const Epi& epi, float* ws, int64_t ws_bytes, cudaStream_t st,
               const char* what) {
  if (PQ % 4 || nseg < 1 || nseg > kMaxSeg) return -1;
  ActMaps amaps{};
  Work w{};
  w.nseg = nseg;
  int kbs = 0;
  for (int i = 0; i < nseg; ++i) {
    if ((reinterpret_cast<uintptr_t>(act[i]) & 15) || kseg[i] < 1) return -1;
    if (!make_act_map(&amaps.m[i], act[i], PQ, kseg[i], imgs)) return -1;
    w.seg_kb[i] = kbs;
    kbs += (kseg[i] + BK - 1) / BK;
  }
  for (int i = nseg; i <= kMaxSeg; ++i) w.seg_kb[i] = kbs;
  const int K = kbs * BK;
  if (nseg == 1) {
    if (kseg[0] < 8) return -1;
  }
  w.PQ = PQ;
  w.tiles_img = (PQ + BM - 1) / BM;
  w.N_img = imgs;
  w.Nout = Nout;
  w.K = nseg == 1 ? kseg[0] : K;
  w.BN = pick_bn(Nout, w.ntiles);
  w.nkb = kbs;
  w.nacc = 2;
  w.b_bytes = 2 * w.BN * 128;
  w.stage_bytes = 2 * kABytes + w.b_bytes;
  const int smem_cap = 227 * 1024;
  const int tail = 1024 + (3 * kMaxStages + 4) * 8 + 64;
  // narrow outputs (BN <= 64): two CTAs per SM, each with half the TMEM and
  // shared memory -- two MMA issuers and two stage pipelines per SM for the
  // issue- and round-trip-latency-bound small layers (conv2/3x3_reduce fwd /
  // dgrad 0.089 / 0.084 -> 0.066 / 0.063 ms, 5x5_reduce layers -10%)
#ifndef TC4_PAIR_MAX_BN
#define TC4_PAIR_MAX_BN 64
#endif
  const bool pair = w.BN <= TC4_PAIR_MAX_BN;
  const int cap = pair ? 113 * 1024 : smem_cap;
  w.tmem_cols = pair ? 256 : 512;
  // separate small-term accumulator where two 2*BN-column buffers fit the
  // CTA's TMEM (BN <= 64 paired, BN <= 128 alone); PURINE_B200_SACC=0 disables
  w.sacc = (2 * 2 * w.BN <= w.tmem_cols && tc4_sacc_enabled()) ? 1 : 0;
  w.accw = w.sacc ? 2 * w.BN : w.BN;
  w.nst = std::min(kMaxStages, (cap - tail) / w.stage_bytes);
  if (w.nst < 2) return -1;
  const int64_t pack_bytes = (int64_t)w.ntiles * w.nkb * w.b_bytes;
  const int64_t pack_aligned = (pack_bytes + 1023) / 1024 * 1024;
  if (!ws || ws_bytes < pack_aligned) return -1;
  uint8_t* bpack = reinterpret_cast<uint8_t*>(ws);
  float* part_ws = reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(ws) + pack_aligned);
  const int64_t part_bytes = ws_bytes - pack_aligned;
  const int M = imgs * PQ;

  launch_pack_b(lbp, Nout, w.K, w.BN, w.nkb, w.ntiles, bpack, st);
  if (int rc = check_launch(what)) return rc;

  const int sms = gemm_sm_budget();
  w.splits = 1;
  const int64_t tiles = (int64_t)imgs * w.tiles_img * w.ntiles;
#ifndef TC4_NOSPLIT_MIN_TILES
#define TC4_NOSPLIT_MIN_TILES 1000000
#endif
  if (tiles < sms && tiles < TC4_NOSPLIT_MIN_TILES) {
    const int64_t want = sms / tiles;
    const int64_t by_k = w.nkb / 2;
    const int64_t by_ws = part_bytes / ((int64_t)M * Nout * 4);
    w.splits = (int)std::max<int64_t>(1, std::min(std::min(want, by_k),
                                                  std::min<int64_t>(by_ws, 256)));
  }
  w.kbps = (w.nkb + w.splits - 1) / w.splits;
  w.splits = (w.nkb + w.kbps - 1) / w.kbps;
  w.units = (int)(tiles * w.splits);

  static bool configured = false;
  if (!configured) {
    BF_CUDA(cudaFuncSetAttribute(tc4_kernel<Epi>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 smem_cap),
            "tc4 smem attribute");
    configured = true;
  }
  // >= 120 KB keeps one CTA (one 512-column TMEM allocation) per SM; a pair
  // CTA takes >= 109 KB so two fit an SM but none shares one with a 512-column
  // engine v2 / v4 CTA (whose allocation would stall behind it)
  const int smem = std::max(tail + w.nst * w.stage_bytes, (pair ? 109 : 120) << 10);
  const int grid = std::min(w.units, pair ? 2 * sms : sms);
  EpiPartial part{part_ws, M, Nout};
  tc4_kernel<Epi><<<grid, kThreads, smem, st>>>(amaps, w, bpack, epi, part);
  if (int rc = check_launch(what)) return rc;
  if (w.splits > 1) {
    splitk_reduce<Epi>(part_ws, w.splits, M, Nout, epi, st);
    return check_launch(what);
  }
  return 0;
}

template <class LBP, class Epi>
int launch(const float* act, int imgs, int K, int PQ, int Nout, const LBP& lbp, const Epi& epi,
           float* ws, int64_t ws_bytes, cudaStream_t st, const char* what) {
  return launch_seg(1, &act, &K, imgs, PQ, Nout, lbp, epi, ws, ws_bytes, st, what);
}

struct LdW1x1 {  // fwd: B(n = kout, k = c) = w[kout][c]
  const float* w;
  int C;
  __device__ __forceinline__ float operator()(int n, int k) const {
    return w[(int64_t)n * C + k];
  }
};
struct LdW1x1Cat {  // grouped fwd: B(n, k) = w[s][n - start[s]][k], n in segment s
  const float* w[kMaxSeg];
  int start[kMaxSeg + 1];
  int nseg, C;
  __device__ __forceinline__ float operator()(int n, int k) const {
    int s = 0;
#pragma unroll
    for (int i = 1; i < kMaxSeg; ++i) s += (i < nseg && n >= start[i]) ? 1 : 0;
    return w[s][(int64_t)(n - start[s]) * C + k];
  }
};
struct LdW1x1TCat {  // grouped dgrad: B(n = c, k) = w[s][k - kstart[s]][c], zero in the padding
  const float* w[kMaxSeg];
  int kstart[kMaxSeg + 1];  // 32-aligned segment starts in the padded K
  int kout[kMaxSeg];
  int nseg, C;
  __device__ __forceinline__ float operator()(int n, int k) const {
    int s = 0;
#pragma unroll
    for (int i = 1; i < kMaxSeg; ++i) s += (i < nseg && k >= kstart[i]) ? 1 : 0;
    const int kk = k - kstart[s];
    return kk < kout[s] ? w[s][(int64_t)kk * C + n] : 0.f;
  }
};
struct LdW1x1T {  // dgrad: B(n = c, k = kout) = w[kout][c]
  const float* w;
  int C;
  __device__ __forceinline__ float operator()(int n, int k) const {
    return w[(int64_t)k * C + n];
  }
};

}  // namespace tc4

static bool tc4_eligible(const ConvShape& g) {
  return g.R == 1 && g.S == 1 && g.stride == 1 && g.pad == 0 && g.P == g.H && g.Q == g.W &&
         (g.H * g.W) % 4 == 0;
}

int tc4_conv_fwd(const ConvShape& g, const float* x, const float* w, const EpiNCHW& epi,
                 float* ws, int64_t ws_bytes, cudaStream_t st, const char* what) {
  if (!tc4_eligible(g)) return -1;
  return tc4::launch(x, g.N, g.C, g.H * g.W, g.K, tc4::LdW1x1{w, g.C}, epi, ws, ws_bytes, st,
                     what);
}

int tc4_conv_fwd_group(const float* x, int N, int C, int HW, int nseg, const float* const* w,
                       const int* kout, const EpiNCHWSeg& epi, float* ws, int64_t ws_bytes,
                       cudaStream_t st, const char* what) {
  if (nseg < 1 || nseg > kMaxSeg || HW % 4) return -1;
  tc4::LdW1x1Cat lb{};
  lb.nseg = nseg;
  lb.C = C;
  int n = 0;
  for (int i = 0; i < nseg; ++i) {
    lb.w[i] = w[i];
    lb.start[i] = n;
    n += kout[i];
  }
  lb.start[nseg] = n;
  for (int i = nseg + 1; i <= kMaxSeg; ++i) lb.start[i] = n;
  return tc4::launch(x, N, C, HW, n, lb, epi, ws, ws_bytes, st, what);
}

int tc4_conv_dgrad_group(int N, int C, int HW, int nseg, const float* const* dy,
                         const float* const* w, const int* kout, const EpiNCHW& epi, float* ws,
                         int64_t ws_bytes, cudaStream_t st, const char* what) {
  if (nseg < 1 || nseg > kMaxSeg || HW % 4) return -1;
  tc4::LdW1x1TCat lb{};
  lb.nseg = nseg;
  lb.C = C;
  int k = 0;
  for (int i = 0; i < nseg; ++i) {
    lb.w[i] = w[i];
    lb.kout[i] = kout[i];
    lb.kstart[i] = k;
    k += (kout[i] + tc4::BK - 1) / tc4::BK * tc4::BK;
  }
  for (int i = nseg; i <= kMaxSeg; ++i) lb.kstart[i] = k;
  return tc4::launch_seg(nseg, dy, kout, N, HW, C, lb, epi, ws, ws_bytes, st, what);
}

int tc4_conv_dgrad(const ConvShape& g, const float* dy, const float* w, const EpiNCHW& epi,
                   float* ws, int64_t ws_bytes, cudaStream_t st, const char* what) {
  if (!tc4_eligible(g)) return -1;
  return tc4::launch(dy, g.N, g.K, g.H * g.W, g.C, tc4::LdW1x1T{w, g.C}, epi, ws, ws_bytes, st,
                     what);
}

}  // namespace bf
