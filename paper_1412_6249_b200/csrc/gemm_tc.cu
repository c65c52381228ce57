// tcgen05 implicit-GEMM engine, fp32-accurate via split TF32 (3xTF32).
//
//   D[m][n] = sum_k A(m,k) B(n,k)          (gemm_common.cuh explains the mapping
//                                           of conv fwd/dgrad/wgrad and fc onto it)
//
// Each fp32 operand x is split into big = TF32 round-to-nearest of x and
// small = TF32(x - big); the tensor core accumulates big*big + big*small +
// small*big into an fp32 TMEM accumulator.  The dropped small*small term and
// the rounding of small are ~2^-22 relative, so the result is within a few
// fp32 ulps of an fp32 GEMM (SURVEY.md finding 7: 1xTF32 misses the 1e-4
// contract at GoogLeNet shapes, 3xTF32 passes).
//
// CTA = 8 producer warps + 1 MMA warp.  Producers gather the operand tiles
// straight from the NCHW tensors (implicit GEMM: no materialised im2col),
// split them and store big/small into 128B-swizzled K-major shared-memory
// tiles (the canonical UMMA SWIZZLE_128B layout, so both the gather stores and
// the tensor-core reads are bank-conflict free); one elected thread of the
// MMA warp issues tcgen05.mma (M=128, N=BN, K=8 per instruction, 3 per k-step)
// from shared-memory descriptors into TMEM and releases each stage with
// tcgen05.commit on an mbarrier; after the last k-block the producers turn
// into the epilogue: tcgen05.ld TMEM -> registers -> coalesced NCHW stores
// (bias fused).  Split-K over gridDim.z writes fp32 partials reduced in a fixed
// order (deterministic).
#include "gemm_common.cuh"
#include "gemm_engines.cuh"

namespace bf {
namespace tc {

constexpr int BM = 128;
constexpr int BK = 32;  // fp32 elements per tile row = 128 bytes = one swizzle atom row
constexpr int kProducerWarps = 8;
constexpr int kProducers = kProducerWarps * 32;
constexpr int kThreads = kProducers + 32;  // + MMA warp
constexpr int kInvalid = -30000;

struct __align__(8) RowInfo {
  int off;
  short h, w;
};

// ---- loaders: separable form  element(row,k) = ptr[row.off + k.off] if in bounds ----
//   in bounds <=> (unsigned)(row.h + k.h) < Hb && (unsigned)(row.w + k.w) < Wb

template <class L>
struct Sep;

template <>
struct Sep<LdFwdX> {  // row = (n,p,q), k = (c,r,s)
  static constexpr bool kMContig = true;
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
  __device__ static int hb(const LdFwdX& l) { return l.g.H; }
  __device__ static int wb(const LdFwdX& l) { return l.g.W; }
  __device__ static const float* ptr(const LdFwdX& l) { return l.x; }
};

template <>
struct Sep<LdDgradDY> {  // stride 1 only: row = (n,h,w), k = (kout,r,s)
  static constexpr bool kMContig = true;
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
  __device__ static int hb(const LdDgradDY& l) { return l.g.P; }
  __device__ static int wb(const LdDgradDY& l) { return l.g.Q; }
  __device__ static const float* ptr(const LdDgradDY& l) { return l.dy; }
};

template <>
struct Sep<LdDgradW> {  // row = c, k = (kout,r,s)
  static constexpr bool kMContig = false;
  __device__ static RowInfo row(const LdDgradW& l, int c) { return {c * l.g.R * l.g.S, 0, 0}; }
  __device__ static RowInfo kin(const LdDgradW& l, int k) {
    int RS = l.g.R * l.g.S;
    int ko = k / RS, rs = k - ko * RS;
    return {ko * l.g.C * RS + rs, 0, 0};
  }
  __device__ static int hb(const LdDgradW&) { return 0x7fffffff; }
  __device__ static int wb(const LdDgradW&) { return 0x7fffffff; }
  __device__ static const float* ptr(const LdDgradW& l) { return l.w; }
};

template <>
struct Sep<LdWgradX> {  // row = (c,r,s), k = (n,p,q)
  static constexpr bool kMContig = false;
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
  __device__ static int hb(const LdWgradX& l) { return l.g.H; }
  __device__ static int wb(const LdWgradX& l) { return l.g.W; }
  __device__ static const float* ptr(const LdWgradX& l) { return l.x; }
};

template <>
struct Sep<LdWgradDY> {  // row = kout, k = (n,pq)
  static constexpr bool kMContig = false;
  __device__ static RowInfo row(const LdWgradDY& l, int ko) { return {ko * l.g.P * l.g.Q, 0, 0}; }
  __device__ static RowInfo kin(const LdWgradDY& l, int k) {
    int PQ = l.g.P * l.g.Q;
    int n = k / PQ, pq = k - n * PQ;
    return {n * l.g.K * PQ + pq, 0, 0};
  }
  __device__ static int hb(const LdWgradDY&) { return 0x7fffffff; }
  __device__ static int wb(const LdWgradDY&) { return 0x7fffffff; }
  __device__ static const float* ptr(const LdWgradDY& l) { return l.dy; }
};

template <>
struct Sep<LdRowK> {
  static constexpr bool kMContig = false;
  __device__ static RowInfo row(const LdRowK& l, int r) { return {(int)(r * l.ld), 0, 0}; }
  __device__ static RowInfo kin(const LdRowK&, int k) { return {k, 0, 0}; }
  __device__ static int hb(const LdRowK&) { return 0x7fffffff; }
  __device__ static int wb(const LdRowK&) { return 0x7fffffff; }
  __device__ static const float* ptr(const LdRowK& l) { return l.p; }
};

template <>
struct Sep<LdColK> {
  static constexpr bool kMContig = true;
  __device__ static RowInfo row(const LdColK&, int r) { return {r, 0, 0}; }
  __device__ static RowInfo kin(const LdColK& l, int k) { return {(int)(k * l.ld), 0, 0}; }
  __device__ static int hb(const LdColK&) { return 0x7fffffff; }
  __device__ static int wb(const LdColK&) { return 0x7fffffff; }
  __device__ static const float* ptr(const LdColK& l) { return l.p; }
};

// ---- PTX wrappers -----------------------------------------------------------

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  uint32_t addr = smem_u32(bar);
  asm volatile(
      "{\n\t.reg .pred P1;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@!P1 bra WAIT_%=;\n\t}" ::"r"(addr),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ void fence_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}

__device__ __forceinline__ void tc_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_u32(bar))
               : "memory");
}

__device__ __forceinline__ void tc_mma_tf32(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc,
                                            uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}

__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&v)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
        "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]),
        "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

__device__ __forceinline__ void named_sync(int id, int count) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(count) : "memory");
}

// K-major SWIZZLE_128B UMMA shared-memory descriptor (sm_100 "version 1")
__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)1 << 16;                    // LBO (unused for swizzled K-major) = 16 B
  d |= (uint64_t)(1024 >> 4) << 32;          // SBO: 8-row group stride = 1024 B
  d |= (uint64_t)1 << 46;                    // descriptor version (sm_100)
  d |= (uint64_t)2 << 61;                    // layout: SWIZZLE_128B
  return d;
}

// instruction descriptor: D=f32, A=B=tf32, both K-major, M=128, N=bn
__host__ __device__ constexpr uint32_t tf32_idesc(int bn) {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(bn >> 3) << 17) |
         ((uint32_t)(BM >> 4) << 24);
}

__device__ __forceinline__ float to_tf32_rna(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}

// big = round-to-nearest TF32 of x; small = TF32(x - big), |small| <= 2^-11 |x|;
// big*big + big*small + small*big then misses x*y by at most ~2^-21 |x y|
__device__ __forceinline__ void split_tf32(float x, float& big, float& small) {
  big = to_tf32_rna(x);
  small = to_tf32_rna(x - big);
}

// byte offset of 16B chunk `c` of row `r` in a 128B-swizzled tile
__device__ __forceinline__ uint32_t sw_off(int r, int c) {
  return (uint32_t)(r * 128 + (((c ^ r) & 7) << 4));
}

// (row, 16B chunk) handled by producer thread t for its e-th chunk of an R-row tile
template <bool kMContig, int E, int R>
__device__ __forceinline__ void chunk_of(int t, int e, int& r, int& c) {
  if (kMContig) {  // consecutive lanes -> consecutive rows (pixel-contiguous operands)
    r = t % R;
    c = (t / R) * E + e;
  } else {         // 8 lanes per row -> 128 contiguous bytes along K
    c = t & 7;
    r = (t >> 3) + 32 * e;
  }
}

template <bool kMContig, int E, int R>
__device__ __forceinline__ void gather(int t, const float* __restrict__ p, const RowInfo* rows,
                                       const RowInfo* ks, unsigned hb, unsigned wb,
                                       float (&v)[E][4]) {
#pragma unroll
  for (int e = 0; e < E; ++e) {
    int r, c;
    chunk_of<kMContig, E, R>(t, e, r, c);
    const RowInfo ri = rows[r];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const RowInfo ki = ks[c * 4 + j];
      bool ok = (unsigned)(ri.h + ki.h) < hb && (unsigned)(ri.w + ki.w) < wb;
      v[e][j] = ok ? __ldg(p + (ri.off + ki.off)) : 0.f;
    }
  }
}

template <bool kMContig, int E, int R>
__device__ __forceinline__ void store_split(int t, const float (&v)[E][4], uint8_t* big,
                                            uint8_t* small) {
#pragma unroll
  for (int e = 0; e < E; ++e) {
    int r, c;
    chunk_of<kMContig, E, R>(t, e, r, c);
    float4 bg, sm;
    split_tf32(v[e][0], bg.x, sm.x);
    split_tf32(v[e][1], bg.y, sm.y);
    split_tf32(v[e][2], bg.z, sm.z);
    split_tf32(v[e][3], bg.w, sm.w);
    const uint32_t off = sw_off(r, c);
    *reinterpret_cast<float4*>(big + off) = bg;
    *reinterpret_cast<float4*>(small + off) = sm;
  }
}

template <int BN, int STAGES>
struct Smem {
  static constexpr int kA = BM * BK * 4;  // bytes of one A tile (big or small)
  static constexpr int kB = BN * BK * 4;
  static constexpr int kStage = 2 * kA + 2 * kB;
  static constexpr int kTiles = STAGES * kStage;
  static constexpr int kTables = 2 * STAGES * BK * 8;  // A and B k-tables per stage
  static constexpr int kRows = (BM + BN) * 8;
  static constexpr int kBars = (2 * STAGES + 2) * 8;
  static constexpr int kTotal = 1024 + kTiles + kTables + kRows + kBars + 16;
};

template <class LA, class LB, class Epi, int BN, int STAGES>
__global__ void __launch_bounds__(kThreads, 1)
    tc_gemm_kernel(LA la, LB lb, int M, int N, int K, int kb_per_split, Epi epi, EpiPartial part,
                   int splits) {
  using SA = Sep<LA>;
  using SB = Sep<LB>;
  using L = Smem<BN, STAGES>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* tiles = base;
  RowInfo* ktab = reinterpret_cast<RowInfo*>(base + L::kTiles);      // [STAGES][2][BK]
  RowInfo* rowA = ktab + 2 * STAGES * BK;                             // [BM]
  RowInfo* rowB = rowA + BM;                                          // [BN]
  uint64_t* full = reinterpret_cast<uint64_t*>(rowB + BN);            // [STAGES]
  uint64_t* empty = full + STAGES;                                    // [STAGES]
  uint64_t* done = empty + STAGES;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(done + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int m0 = blockIdx.x * BM, n0 = blockIdx.y * BN;
  const int kb0 = blockIdx.z * kb_per_split;
  const int nkb_total = (K + BK - 1) / BK;
  const int nkb = min(kb_per_split, nkb_total - kb0);
  constexpr uint32_t kTmemCols = BN < 32 ? 32 : BN;

  if (warp == kProducerWarps) {
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
    mbar_init(done, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  // per-row gather info of this tile
  for (int i = threadIdx.x; i < BM + BN; i += kThreads) {
    if (i < BM) {
      int m = m0 + i;
      rowA[i] = m < M ? SA::row(la, m) : RowInfo{0, (short)kInvalid, (short)kInvalid};
    } else {
      int n = n0 + i - BM;
      rowB[i - BM] = n < N ? SB::row(lb, n) : RowInfo{0, (short)kInvalid, (short)kInvalid};
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp < kProducerWarps) {
    // ===================== producers: gather -> split -> swizzled smem =====================
    const float* pa = SA::ptr(la);
    const float* pb = SB::ptr(lb);
    const unsigned hbA = (unsigned)SA::hb(la), wbA = (unsigned)SA::wb(la);
    const unsigned hbB = (unsigned)SB::hb(lb), wbB = (unsigned)SB::wb(lb);
    const int t = threadIdx.x;
    for (int i = 0; i < nkb; ++i) {
      const int stage = i % STAGES;
      const uint32_t phase = (i / STAGES) & 1;
      const int kbase = (kb0 + i) * BK;
      RowInfo* kA = ktab + (stage * 2 + 0) * BK;
      RowInfo* kB = ktab + (stage * 2 + 1) * BK;
      if (t < BK) {
        int k = kbase + t;
        kA[t] = k < K ? SA::kin(la, k) : RowInfo{0, (short)kInvalid, (short)kInvalid};
      } else if (t < 2 * BK) {
        int k = kbase + t - BK;
        kB[t - BK] = k < K ? SB::kin(lb, k) : RowInfo{0, (short)kInvalid, (short)kInvalid};
      }
      named_sync(1, kProducers);
      mbar_wait(&empty[stage], phase ^ 1);
      uint8_t* st = tiles + stage * L::kStage;
      uint8_t* a_big = st;
      uint8_t* a_small = st + L::kA;
      uint8_t* b_big = st + 2 * L::kA;
      uint8_t* b_small = st + 2 * L::kA + L::kB;

      // all loads of both operands are issued before the first use so that
      // ~(BM+BN)*BK/256 gathers per thread are in flight at once
      constexpr int EA = BM * 8 / kProducers, EB = BN * 8 / kProducers;
      float va[EA][4], vb[EB][4];
      gather<SA::kMContig, EA, BM>(t, pa, rowA, kA, hbA, wbA, va);
      gather<SB::kMContig, EB, BN>(t, pb, rowB, kB, hbB, wbB, vb);
      store_split<SA::kMContig, EA, BM>(t, va, a_big, a_small);
      store_split<SB::kMContig, EB, BN>(t, vb, b_big, b_small);
      fence_async_smem();
      mbar_arrive(&full[stage]);
    }
  } else if (lane == 0) {
    // ===================== MMA issuer: one thread =====================
    constexpr uint32_t idesc = tf32_idesc(BN);
    for (int i = 0; i < nkb; ++i) {
      const int stage = i % STAGES;
      const uint32_t phase = (i / STAGES) & 1;
      mbar_wait(&full[stage], phase);
      tc_fence_after();
      const uint32_t st = smem_u32(tiles + stage * L::kStage);
      const uint32_t a_big = st, a_small = st + L::kA;
      const uint32_t b_big = st + 2 * L::kA, b_small = st + 2 * L::kA + L::kB;
#pragma unroll
      for (int ks = 0; ks < BK / 8; ++ks) {
        const uint32_t koff = ks * 32;  // 8 tf32 = 32 bytes along K inside the swizzle atom
        uint64_t dab = sw128_desc(a_big + koff), das = sw128_desc(a_small + koff);
        uint64_t dbb = sw128_desc(b_big + koff), dbs = sw128_desc(b_small + koff);
        uint32_t acc = (i > 0 || ks > 0) ? 1u : 0u;
        tc_mma_tf32(tmem, das, dbb, idesc, acc);
        tc_mma_tf32(tmem, dab, dbs, idesc, 1u);
        tc_mma_tf32(tmem, dab, dbb, idesc, 1u);
      }
      tc_commit(&empty[stage]);
    }
    tc_commit(done);
  }

  // ===================== epilogue: TMEM -> registers -> global =====================
  if (warp < kProducerWarps) {
    mbar_wait(done, 0);
    tc_fence_after();
    const int q = warp & 3;            // TMEM lane quarter this warp may access
    const int half = warp >> 2;        // which half of the columns
    const int m = m0 + q * 32 + lane;
    constexpr int kCols = BN / 2;
#pragma unroll 1
    for (int c0 = half * kCols; c0 < half * kCols + kCols; c0 += 16) {
      uint32_t v[16];
      tmem_ld16(tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)c0, v);
      if (m < M) {
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          int n = n0 + c0 + j;
          if (n < N) {
            if (splits > 1)
              part(blockIdx.z, m, n, __uint_as_float(v[j]));
            else
              epi(m, n, __uint_as_float(v[j]));
          }
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == kProducerWarps) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                 "r"(kTmemCols));
  }
}

template <class LA, class LB, class Epi, int BN, int STAGES>
int launch(const LA& la, const LB& lb, int M, int N, int K, const Epi& epi, float* ws,
           int64_t ws_bytes, cudaStream_t st, const char* what) {
  using L = Smem<BN, STAGES>;
  auto kern = tc_gemm_kernel<LA, LB, Epi, BN, STAGES>;
  static bool configured = false;
  if (!configured) {
    BF_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, L::kTotal),
            "tc_gemm smem attribute");
    configured = true;
  }
  const int nkb = (K + BK - 1) / BK;
  int splits = choose_splits(M, N, K, BM, BN, 8 * BK, ws ? ws_bytes : 0);
  int kbps = (nkb + splits - 1) / splits;
  splits = (nkb + kbps - 1) / kbps;
  dim3 grid((M + BM - 1) / BM, (N + BN - 1) / BN, splits);
  EpiPartial part{ws, M, N};
  kern<<<grid, kThreads, L::kTotal, st>>>(la, lb, M, N, K, kbps, epi, part, splits);
  if (int rc = check_launch(what)) return rc;
  if (splits > 1) {
    splitk_reduce<Epi>(ws, splits, M, N, epi, st);
    return check_launch(what);
  }
  return 0;
}

template <class L>
inline bool separable(const L&) {
  return true;
}
template <>
inline bool separable<LdDgradDY>(const LdDgradDY& l) {
  return l.g.stride == 1;
}

}  // namespace tc

template <class LA, class LB, class Epi>
int tc_gemm(const LA& la, const LB& lb, int M, int N, int K, const Epi& epi, float* ws,
            int64_t ws_bytes, cudaStream_t st, const char* what) {
  if (!tc::separable(la) || !tc::separable(lb)) return -1;
  if (M < 64 || K < 16) return -1;  // tiny problems: SIMT engine
  if (N <= 64) return tc::launch<LA, LB, Epi, 64, 4>(la, lb, M, N, K, epi, ws, ws_bytes, st, what);
  return tc::launch<LA, LB, Epi, 128, 3>(la, lb, M, N, K, epi, ws, ws_bytes, st, what);
}

#define BF_TC_INST(LA, LB, EPI) \
  template int tc_gemm<LA, LB, EPI>(const LA&, const LB&, int, int, int, const EPI&, float*, \
                                    int64_t, cudaStream_t, const char*);
BF_TC_INST(LdFwdX, LdRowK, EpiNCHW)
BF_TC_INST(LdDgradDY, LdDgradW, EpiNCHW)
BF_TC_INST(LdWgradX, LdWgradDY, EpiT)
BF_TC_INST(LdColK, LdRowK, EpiT)
BF_TC_INST(LdRowK, LdRowK, EpiT)
BF_TC_INST(LdColK, LdColK, EpiT)

}  // namespace bf

extern "C" int bf_has_tcgen05(void) { return 1; }
