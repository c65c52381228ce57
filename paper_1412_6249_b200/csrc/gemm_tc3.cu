// tcgen05 implicit-GEMM engine v3: halo-staged stride-1 R x S convolutions
// (conv forward and data gradient, 3xTF32).
//
// Engine v2 (gemm_tc2.cu) gathers the im2col operand element by element: a
// 3x3 layer loads, splits and stores every input value 9 times (25 for 5x5).
// v3 removes the duplication with a padded-grid formulation:
//
//  * Output pixels are enumerated on the zero-padded input grid
//    (Hp = H + 2 pad, Wp = W + 2 pad): row o = (n*Hp + p)*Wp + q.  Filter tap
//    (r, s) of row o then reads padded-grid row o + r*Wp + s, for every o: a
//    constant shift.  Rows with p >= P or q >= Q are computed and discarded
//    (the epilogue skips them; 7-40% extra MMA on the small late layers).
//  * Per 32-channel block, the producers stage the tile's rows plus the halo
//    (BM + (R-1)*Wp + (S-1) padded rows x 32 channels) ONCE into shared
//    memory, already split into TF32 big/small images (128-byte rows,
//    16-byte chunks XOR-swizzled by row so both the staging stores and the
//    per-tap row reads are bank-conflict free).
//  * For each of the R*S taps, each producer thread copies its pixel row's
//    shifted 16 channels (4 x 16-byte loads per image) into the TMEM A ring
//    with tcgen05.st; the MMA warp issues the same 3xTF32 tcgen05.mma
//    sequence as v2 against the tap's pre-packed weight tile (bulk TMA).
//
// So per input element: one global load and one split per channel block,
// and per tap only shared-memory reads -- the im2col duplication costs LDS
// bandwidth instead of gather + split instructions.  The data gradient of a
// stride-1 convolution is the same operation on dY with pad' = R-1-pad and
// the flipped, transposed filter (ops.py:300-343 restated by the oracle as
// oracle/kernels.py conv2d_backward_data).
//
// Measured (GoogLeNet batch 128, tools/conv_bench.py): v3 is NOT faster than
// v2.  The large 3x3 layers already run v2 at 150-180 TFLOP/s, close to the
// 3xTF32 tensor ceiling, so removing gather work cannot help them; on the small
// late layers the discarded border rows (up to 60% on 7x7 maps) and the
// serial per-block staging cost more than they save.  v3 therefore stays
// opt-in (bf_set_gemm_engine(3)) and covered by the GPU parity tests.
#include <algorithm>

#include "gemm_common.cuh"
#include "gemm_engines.cuh"
#include "tc_ptx.cuh"

namespace bf {
namespace tc3 {

using namespace tcu;

constexpr int BK = 32;  // channels per block = one 128-byte smem row
constexpr int STAGES = 4;
constexpr int kProducerWarps = 8;
constexpr int kProducers = kProducerWarps * 32;
constexpr int kEpiWarps = 8;
constexpr int kMmaWarp = kProducerWarps;
constexpr int kAllThreads = (kProducerWarps + 1 + kEpiWarps) * 32;
constexpr uint32_t kTmemCols = 512;
constexpr uint32_t kAColBase = 256;

// the implicit GEMM's input (x for fwd, dy for dgrad) and its padded grid
struct Halo {
  const float* in;  // [N][Cin][Hin][Win]
  int N, Cin, Hin, Win, pad;
  int Hp, Wp, R, S, P, Q;  // padded grid; outputs P = Hp-R+1, Q = Wp-S+1
  int ncb, rows;           // channel blocks; staged rows per tile (BM + halo)
};

struct Work {
  int Mp, Nout, BN, ntiles, mtiles, nkb, cbps, splits, units, nacc, nst;
};

// fwd: B(n = kout, k') = w[kout][c][tap];  dgrad: B(n = c, k') = w[ko][c][RS-1-tap]
// with k' = (cb*RS + tap)*32 + cc and input channel cb*32 + cc
struct LdHaloW {
  const float* w;
  int Cin, Cout, RS;
  bool dgrad;
  __device__ __forceinline__ float operator()(int n, int k) const {
    const int kb = k >> 5, cc = k & 31;
    const int cb = kb / RS, tap = kb - cb * RS;
    const int c = cb * 32 + cc;
    if (c >= Cin) return 0.f;
    if (!dgrad) return w[((int64_t)n * Cin + c) * RS + tap];
    return w[((int64_t)c * Cout + n) * RS + (RS - 1 - tap)];
  }
};

__device__ __forceinline__ void unit_coords(const Work& w, int u, int& mt, int& nt, int& sp) {
  sp = u % w.splits;
  int r = u / w.splits;
  nt = r % w.ntiles;
  mt = r / w.ntiles;
}

__device__ __forceinline__ uint32_t halo_off(int j, int chunk) {
  return (uint32_t)(j * 128 + (((chunk ^ j) & 7) << 4));
}

// stage padded-grid rows [o0, o0 + rows) x channels [cb*32, +32) as TF32 big/small
__device__ __forceinline__ void stage_halo(const Halo& h, int o0, int cb, uint8_t* big,
                                           uint8_t* small, int t) {
  const int HW = h.Hin * h.Win;
  const int plane = h.Hp * h.Wp;
  const int Mp = h.N * plane;
  const int cbase = cb * BK;
  const int nch = min(BK, h.Cin - cbase);
  for (int j = t; j < h.rows; j += kProducers) {
    const int o = o0 + j;
    const float* src = nullptr;
    if (o < Mp) {
      const int n = o / plane, rem = o - n * plane;
      const int hp = rem / h.Wp, wp = rem - hp * h.Wp;
      const int ih = hp - h.pad, iw = wp - h.pad;
      if ((unsigned)ih < (unsigned)h.Hin && (unsigned)iw < (unsigned)h.Win)
        src = h.in + ((int64_t)n * h.Cin + cbase) * HW + ih * h.Win + iw;
    }
    float v[BK];
#pragma unroll
    for (int c = 0; c < BK; ++c) v[c] = (src && c < nch) ? __ldg(src + (int64_t)c * HW) : 0.f;
#pragma unroll
    for (int q = 0; q < BK / 4; ++q) {
      float4 bg, sm;
      bg.x = to_tf32_rna(v[4 * q + 0]); sm.x = to_tf32_rna(v[4 * q + 0] - bg.x);
      bg.y = to_tf32_rna(v[4 * q + 1]); sm.y = to_tf32_rna(v[4 * q + 1] - bg.y);
      bg.z = to_tf32_rna(v[4 * q + 2]); sm.z = to_tf32_rna(v[4 * q + 2] - bg.z);
      bg.w = to_tf32_rna(v[4 * q + 3]); sm.w = to_tf32_rna(v[4 * q + 3] - bg.w);
      const uint32_t off = halo_off(j, q);
      *reinterpret_cast<float4*>(big + off) = bg;
      *reinterpret_cast<float4*>(small + off) = sm;
    }
  }
}

template <class Epi>
__global__ void __launch_bounds__(kAllThreads, 1)
    tc3_kernel(Halo h, Work w, const uint8_t* __restrict__ bpack, Epi epi, EpiPartial part) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  const int BN = w.BN;
  const int stage_bytes = 2 * BN * 128;
  const int RS = h.R * h.S;
  uint8_t* tiles = base;
  uint8_t* hbig = base + w.nst * stage_bytes;
  uint8_t* hsmall = hbig + h.rows * 128;
  uint64_t* full = reinterpret_cast<uint64_t*>(hsmall + h.rows * 128);
  uint64_t* empty = full + STAGES;
  uint64_t* acc_full = empty + STAGES;
  uint64_t* acc_empty = acc_full + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 2);

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
    for (int b = 0; b < 2; ++b) {
      mbar_init(&acc_full[b], 1);
      mbar_init(&acc_empty[b], kEpiWarps * 32);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp < kProducerWarps) {
    // ======================= producers =======================
    const int t = threadIdx.x;
    const int q = warp & 3;
    const int chunk0 = (warp >> 2) * 4;  // 16-channel half of the block: chunks chunk0..+3
    const int row = q * 32 + lane;       // this thread's TMEM lane = tile row
    const uint32_t lane_addr = tmem + ((uint32_t)(q * 32) << 16);
    int it = 0;
    for (int u = blockIdx.x; u < w.units; u += gridDim.x) {
      int mt, nt, sp;
      unit_coords(w, u, mt, nt, sp);
      const int cb0 = sp * w.cbps;
      const int cb1 = min(h.ncb, cb0 + w.cbps);
      for (int cb = cb0; cb < cb1; ++cb) {
        named_sync(1, kProducers);  // every thread is done reading the previous block
        stage_halo(h, mt * BM, cb, hbig, hsmall, t);
        named_sync(1, kProducers);
        for (int tap = 0; tap < RS; ++tap) {
          const int r = tap / h.S, s = tap - r * h.S;
          const int j = row + r * h.Wp + s;
          float big[16], small[16];
#pragma unroll
          for (int c4 = 0; c4 < 4; ++c4) {
            const uint32_t off = halo_off(j, chunk0 + c4);
            const float4 b4 = *reinterpret_cast<const float4*>(hbig + off);
            const float4 s4 = *reinterpret_cast<const float4*>(hsmall + off);
            big[4 * c4 + 0] = b4.x; big[4 * c4 + 1] = b4.y;
            big[4 * c4 + 2] = b4.z; big[4 * c4 + 3] = b4.w;
            small[4 * c4 + 0] = s4.x; small[4 * c4 + 1] = s4.y;
            small[4 * c4 + 2] = s4.z; small[4 * c4 + 3] = s4.w;
          }
          const int stage = it % w.nst;
          const uint32_t phase = (it / w.nst) & 1;
          mbar_wait(&empty[stage], phase ^ 1);
          if (t == 0) {
            mbar_expect_tx(&full[stage], (uint32_t)stage_bytes);
            bulk_g2s(smem_u32(tiles + stage * stage_bytes),
                     bpack + ((size_t)nt * w.nkb + cb * RS + tap) * stage_bytes,
                     (uint32_t)stage_bytes, &full[stage]);
          }
          const uint32_t acol = kAColBase + stage * 64 + chunk0 * 4;
          tmem_st16(lane_addr + acol, big);
          tmem_st16(lane_addr + acol + 32, small);
          asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
          tc_fence_before();
          mbar_arrive(&full[stage]);
          ++it;
        }
      }
    }
  } else if (warp == kMmaWarp) {
    // ======================= MMA issuer (as engine v2) =======================
    // whole warp walks the schedule; one elected lane issues (see gemm_tc2.cu)
    {
      const uint32_t idesc = tf32_idesc(BN);
      int it = 0, local = 0;
      for (int u = blockIdx.x; u < w.units; u += gridDim.x, ++local) {
        int mt, nt, sp;
        unit_coords(w, u, mt, nt, sp);
        const int cb0 = sp * w.cbps;
        const int nk = (min(h.ncb, cb0 + w.cbps) - cb0) * RS;
        const int b = local % w.nacc;
        const uint32_t use = local / w.nacc;
        mbar_wait(&acc_empty[b], (use & 1) ^ 1);
        tc_fence_after();
        const uint32_t dacc = tmem + (uint32_t)(b * 128);
        for (int i = 0; i < nk; ++i, ++it) {
          const int stage = it % w.nst;
          const uint32_t phase = (it / w.nst) & 1;
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint32_t bb = smem_u32(tiles + stage * stage_bytes);
          const uint32_t bs = bb + BN * 128;
          const uint32_t ab = tmem + kAColBase + stage * 64;
          if (elect_one()) {
#pragma unroll
            for (int ks = 0; ks < BK / 8; ++ks) {
              const uint64_t dbb = sw128_desc(bb + ks * 32), dbs = sw128_desc(bs + ks * 32);
              const uint32_t a_big = ab + ks * 8, a_small = ab + 32 + ks * 8;
              mma_ts(dacc, a_small, dbb, idesc, (i > 0 || ks > 0) ? 1u : 0u);
              mma_ts(dacc, a_big, dbs, idesc, 1u);
              mma_ts(dacc, a_big, dbb, idesc, 1u);
            }
            tc_commit(&empty[stage]);
          }
          __syncwarp();
        }
        if (elect_one()) tc_commit(&acc_full[b]);
        __syncwarp();
      }
    }
  } else {
    // ======================= epilogue =======================
    const int ew = warp - kMmaWarp - 1;
    const int q = warp & 3;
    const int half = ew >> 2;
    const int plane = h.Hp * h.Wp;
    int local = 0;
    for (int u = blockIdx.x; u < w.units; u += gridDim.x, ++local) {
      int mt, nt, sp;
      unit_coords(w, u, mt, nt, sp);
      const int b = local % w.nacc;
      const uint32_t use = local / w.nacc;
      mbar_wait(&acc_full[b], use & 1);
      tc_fence_after();
      // padded-grid row -> real output pixel (or a discarded border row)
      const int o = mt * BM + q * 32 + lane;
      bool live = o < w.Mp;
      int m = 0;
      if (live) {
        const int n = o / plane, rem = o - n * plane;
        const int p = rem / h.Wp, qq = rem - p * h.Wp;
        live = p < h.P && qq < h.Q;
        m = (n * h.P + p) * h.Q + qq;
      }
      const int n0 = nt * BN;
      const int cols = BN / 2;
      const uint32_t taddr = tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(b * 128);
      const RowPtr rp = live ? (w.splits > 1 ? part.row(sp, m) : epi.row(m)) : RowPtr{nullptr, 0.f};
#pragma unroll 1
      for (int c0 = half * cols; c0 < half * cols + cols; c0 += 16) {
        uint32_t v[16];
        tmem_ld16(taddr + (uint32_t)c0, v);
        if (live) {
          const int nlim = w.Nout - (n0 + c0);
          if (w.splits > 1) {
#pragma unroll
            for (int j = 0; j < 16; ++j)
              if (j < nlim) part.store(rp, n0 + c0 + j, __uint_as_float(v[j]));
          } else {
#pragma unroll
            for (int j = 0; j < 16; ++j)
              if (j < nlim) epi.store(rp, n0 + c0 + j, __uint_as_float(v[j]));
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
                 "r"(kTmemCols));
  }
}

// BN: the whole output-channel extent up to 256 per tile, in multiples of 32
// (the epilogue's two column halves are then multiples of 16)
inline int pick_bn(int N, int& ntiles) {
  ntiles = (N + 255) / 256;
  int per = (N + ntiles - 1) / ntiles;
  return (per + 31) / 32 * 32;
}

int launch(const Halo& h, const LdHaloW& lbp, int Nout, const EpiNCHW& epi, float* ws,
           int64_t ws_bytes, cudaStream_t st, const char* what) {
  const int RS = h.R * h.S;
  Work w{};
  w.Mp = h.N * h.Hp * h.Wp;
  w.Nout = Nout;
  w.BN = pick_bn(Nout, w.ntiles);
  w.nkb = h.ncb * RS;
  w.mtiles = (w.Mp + BM - 1) / BM;
  w.nacc = w.BN <= 128 ? 2 : 1;
  const int64_t stage_bytes = 2LL * w.BN * 128;
  const int smem_cap = 227 * 1024;
  const int tail = 1024 + 16 * 8 + 64;
  const int64_t halo_bytes = 2LL * h.rows * 128;
  w.nst = (int)std::min<int64_t>(STAGES, (smem_cap - tail - halo_bytes) / stage_bytes);
  if (w.nst < 2) return -1;
  const int64_t pack_bytes = (int64_t)w.ntiles * w.nkb * stage_bytes;
  const int64_t pack_aligned = (pack_bytes + 1023) / 1024 * 1024;
  if (!ws || ws_bytes < pack_aligned) return -1;
  uint8_t* bpack = reinterpret_cast<uint8_t*>(ws);
  float* part_ws = reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(ws) + pack_aligned);
  const int64_t part_bytes = ws_bytes - pack_aligned;
  const int Mreal = h.N * h.P * h.Q;

  launch_pack_b(lbp, Nout, w.nkb * BK, w.BN, w.nkb, w.ntiles, bpack, st);
  if (int rc = check_launch(what)) return rc;

  const int sms = gemm_sm_budget();
  w.splits = 1;
  const int64_t tiles = (int64_t)w.mtiles * w.ntiles;
  if (tiles < sms) {  // one wave: split the channel blocks
    const int64_t want = sms / tiles;
    const int64_t by_ws = part_bytes / ((int64_t)Mreal * Nout * 4);
    w.splits = (int)std::max<int64_t>(1, std::min(std::min<int64_t>(want, h.ncb),
                                                  std::min<int64_t>(by_ws, 256)));
  }
  w.cbps = (h.ncb + w.splits - 1) / w.splits;
  w.splits = (h.ncb + w.cbps - 1) / w.cbps;
  w.units = w.mtiles * w.ntiles * w.splits;

  const int smem = tail + (int)(w.nst * stage_bytes + halo_bytes);
  static bool configured = false;
  if (!configured) {
    BF_CUDA(cudaFuncSetAttribute(tc3_kernel<EpiNCHW>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 smem_cap),
            "tc3 smem attribute");
    configured = true;
  }
  const int smem_req = std::max(smem, 120 << 10);  // one CTA (one TMEM allocation) per SM
  const int grid = std::min(w.units, sms);
  EpiPartial part{part_ws, Mreal, Nout};
  tc3_kernel<EpiNCHW><<<grid, kAllThreads, smem_req, st>>>(h, w, bpack, epi, part);
  if (int rc = check_launch(what)) return rc;
  if (w.splits > 1) {
    splitk_reduce<EpiNCHW>(part_ws, w.splits, Mreal, Nout, epi, st);
    return check_launch(what);
  }
  return 0;
}

inline Halo make_halo(const float* in, int N, int Cin, int Hin, int Win, int pad, int R, int S) {
  Halo h;
  h.in = in;
  h.N = N;
  h.Cin = Cin;
  h.Hin = Hin;
  h.Win = Win;
  h.pad = pad;
  h.Hp = Hin + 2 * pad;
  h.Wp = Win + 2 * pad;
  h.R = R;
  h.S = S;
  h.P = h.Hp - R + 1;
  h.Q = h.Wp - S + 1;
  h.ncb = (Cin + BK - 1) / BK;
  h.rows = BM + (R - 1) * h.Wp + (S - 1);
  return h;
}

}  // namespace tc3

// the engine takes stride-1 convolutions with a spatial filter; -1 = not taken
static bool tc3_eligible(const ConvShape& g) {
  return g.stride == 1 && g.R * g.S > 1 && (int64_t)g.N * (g.H + 2 * g.pad) * (g.W + 2 * g.pad) <
                                               (1LL << 31);
}

int tc3_conv_fwd(const ConvShape& g, const float* x, const float* w, const EpiNCHW& epi,
                 float* ws, int64_t ws_bytes, cudaStream_t st, const char* what) {
  if (!tc3_eligible(g)) return -1;
  const tc3::Halo h = tc3::make_halo(x, g.N, g.C, g.H, g.W, g.pad, g.R, g.S);
  if (h.P != g.P || h.Q != g.Q) return -1;
  tc3::LdHaloW lbp{w, g.C, g.K, g.R * g.S, false};
  return tc3::launch(h, lbp, g.K, epi, ws, ws_bytes, st, what);
}

int tc3_conv_dgrad(const ConvShape& g, const float* dy, const float* w, const EpiNCHW& epi,
                   float* ws, int64_t ws_bytes, cudaStream_t st, const char* what) {
  if (!tc3_eligible(g) || g.pad > g.R - 1 || g.pad > g.S - 1 || g.R != g.S) return -1;
  const tc3::Halo h = tc3::make_halo(dy, g.N, g.K, g.P, g.Q, g.R - 1 - g.pad, g.R, g.S);
  if (h.P != g.H || h.Q != g.W) return -1;
  tc3::LdHaloW lbp{w, g.K, g.C, g.R * g.S, true};
  return tc3::launch(h, lbp, g.C, epi, ws, ws_bytes, st, what);
}

}  // namespace bf
