// 3x3 max pooling (stride 1 or 2), staged through shared memory by bulk
// copies: the HBM-bound forward / backward of every GoogLeNet and NIN max
// pool (maxpool_forward / maxpool_backward, oracle/kernels.py:340-379).
//
// Layout: NCHW planes are contiguous, so a chunk of G consecutive planes is
// ONE contiguous range of x (and of dy / y).  A persistent CTA walks its
// chunks through an NS-deep ring of shared-memory stages; one thread issues
// each stage's cp.async.bulk loads (completing on the stage's mbarrier) NS-1
// chunks ahead, so every SM keeps ~64-100 KB of loads in flight (the round-1
// kernels issued 4-byte loads a few rows ahead and reached 2.2-2.4 TB/s).
//
// Forward: a thread walks one output column down a run of RB output rows,
// keeping the three row reductions (first max of the window's 3 columns,
// its flat index) of the current window in registers: S new input rows per
// output (3 shared loads each).  The window result is the first row whose row
// max is strictly greater than the earlier rows' -- exactly the first
// maximum in window raster order with strict '>' from -inf (the oracle's
// scan, NaN and all -inf included).  The argmax mask is written only when
// someone reads it (`mask` may be null): maxpool_backward recomputes it.
//
// Backward (bf_maxpool_bwd_x): the stage holds the chunk's x and dy; phase 1
// recomputes every window's argmax (the forward's walker) into shared memory,
// phase 2 gathers for each input pixel, in window raster order, dy of the
// windows whose argmax it is (bit-exact with the oracle's ordered scatter).
// Stride 1 walks input columns with the 3x3 candidate windows rolling in
// registers; stride 2 tests the <= 2x2 covering windows directly.  With
// relu_from_x the ReLU backward of the operator that produced x is folded in:
// x = relu(a) > 0 <=> a > 0, so dx = x > 0 ? acc : 0 (relu_backward's select).
#include <stdlib.h>

#include <algorithm>

#include "common.cuh"
#include "tc_ptx.cuh"

namespace bf {
namespace pools {

using namespace tcu;

constexpr int kThreads = 512;
constexpr int kMaxStages = 4;

struct Geo {
  int H, W, P, Q, pad;
  int64_t planes;
  int G;            // planes per chunk
  int64_t nchunks;
  int RB;           // output rows per walker run (forward, backward phase 1)
  int runs;         // ceil(P / RB)
  int RBh, hruns;   // backward phase 2 (stride 1): input rows per run, runs
  int NS;           // ring stages
  int stage_floats; // floats per stage (16-byte multiple)
  // exact multiply-shift division (x < 2^31) for the per-item index decode:
  // items per plane (phase 1 / forward), output columns, items per plane
  // (backward phase 2), its inner extent
  uint64_t m_pp1, m_q, m_pp2, m_in2;
  int s_pp1, s_q, s_pp2, s_in2;
  // stride-1 forward over column pairs (Q even): items per plane, pairs per row
  int pairs;  // 0: one column per item
  uint64_t m_pp1p, m_qp;
  int s_pp1p, s_qp;
  // stride-1 backward over input-column pairs (W even)
  int pairs2, RBh2, hruns2;
  uint64_t m_pp2p, m_in2p;
  int s_pp2p, s_in2p;
};

__device__ __forceinline__ int fdiv(int x, uint64_t m, int s) {
  return (int)(((uint64_t)(uint32_t)x * m) >> s);
}

// first maximum of input row h's window columns ws, ws+1, ws+2 (strict '>'
// from -inf; out-of-plane taps never win): value and column offset 0..2
// (-1: none)
__device__ __forceinline__ void row_red(const float* __restrict__ xs, int W, bool rv, int off,
                                        bool c0, bool c1, bool c2, float& m, int& d) {
  const float v0 = (rv && c0) ? xs[off] : -INFINITY;
  const float v1 = (rv && c1) ? xs[off + 1] : -INFINITY;
  const float v2 = (rv && c2) ? xs[off + 2] : -INFINITY;
  m = -INFINITY;
  d = -1;
  if (v0 > m) { m = v0; d = 0; }
  if (v1 > m) { m = v1; d = 1; }
  if (v2 > m) { m = v2; d = 2; }
}

// walk output column pw of one plane over output rows [ph0, ph1); emit(ph, best, arg, li)
// with arg the flat index h*W + w of the window's first maximum (-1: none) and li
// its index 0..8 inside the 3x3 window (row-major)
template <int S, class Emit>
__device__ __forceinline__ void walk_windows(const float* __restrict__ xs, int H, int W, int pad,
                                             int pw, int ph0, int ph1, Emit&& emit) {
  const int ws = pw * S - pad;
  const bool c0 = (unsigned)ws < (unsigned)W, c1 = (unsigned)(ws + 1) < (unsigned)W,
             c2 = (unsigned)(ws + 2) < (unsigned)W;
  float m0, m1, m2;
  int d0, d1, d2;
  int h = ph0 * S - pad;  // top row of the current window
  row_red(xs, W, (unsigned)h < (unsigned)H, h * W + ws, c0, c1, c2, m0, d0);
  row_red(xs, W, (unsigned)(h + 1) < (unsigned)H, (h + 1) * W + ws, c0, c1, c2, m1, d1);
  row_red(xs, W, (unsigned)(h + 2) < (unsigned)H, (h + 2) * W + ws, c0, c1, c2, m2, d2);
  for (int ph = ph0;;) {
    float best = -INFINITY;
    int arg = -1, li = -1;
    if (m0 > best) { best = m0; arg = h * W + ws + d0; li = d0; }
    if (m1 > best) { best = m1; arg = (h + 1) * W + ws + d1; li = 3 + d1; }
    if (m2 > best) { best = m2; arg = (h + 2) * W + ws + d2; li = 6 + d2; }
    emit(ph, best, arg, li);
    if (++ph >= ph1) break;
    h += S;
    if (S == 1) {
      m0 = m1; d0 = d1;
      m1 = m2; d1 = d2;
      row_red(xs, W, (unsigned)(h + 2) < (unsigned)H, (h + 2) * W + ws, c0, c1, c2, m2, d2);
    } else {
      m0 = m2; d0 = d2;
      row_red(xs, W, (unsigned)(h + 1) < (unsigned)H, (h + 1) * W + ws, c0, c1, c2, m1, d1);
      row_red(xs, W, (unsigned)(h + 2) < (unsigned)H, (h + 2) * W + ws, c0, c1, c2, m2, d2);
    }
  }
}

// stride 1, two adjacent output columns pw, pw + 1 (windows a, b over input
// columns ws..ws+2 and ws+1..ws+3): four shared loads and five first-max folds
// per new row instead of six and six.  The folds are seeded with -inf, so the
// result is the first maximum in window raster order with strict '>', exactly
// walk_windows' (NaN never wins, ties keep the earlier tap).
struct Mx {
  float m;
  int d;  // column offset inside the window, -1: none
};
__device__ __forceinline__ void fold(Mx& a, float v, int d) {
  if (v > a.m) { a.m = v; a.d = d; }
}
template <class Emit>
__device__ __forceinline__ void walk_pair(const float* __restrict__ xs, int H, int W, int pad,
                                          int pw, int ph0, int ph1, Emit&& emit) {
  const int ws = pw - pad;
  const bool c0 = (unsigned)ws < (unsigned)W, c1 = (unsigned)(ws + 1) < (unsigned)W,
             c2 = (unsigned)(ws + 2) < (unsigned)W, c3 = (unsigned)(ws + 3) < (unsigned)W;
  auto row = [&](int h, Mx& ra, Mx& rb) {
    const bool rv = (unsigned)h < (unsigned)H;
    const int off = h * W + ws;
    const float v0 = (rv && c0) ? xs[off] : -INFINITY;
    const float v1 = (rv && c1) ? xs[off + 1] : -INFINITY;
    const float v2 = (rv && c2) ? xs[off + 2] : -INFINITY;
    const float v3 = (rv && c3) ? xs[off + 3] : -INFINITY;
    Mx p{-INFINITY, -1};  // first max of columns ws+1, ws+2 (offsets 0, 1 from ws+1)
    fold(p, v1, 0);
    fold(p, v2, 1);
    ra = Mx{-INFINITY, -1};
    fold(ra, v0, 0);
    if (p.m > ra.m) { ra.m = p.m; ra.d = p.d + 1; }
    rb = p;
    fold(rb, v3, 2);
  };
  Mx a0, a1, a2, b0, b1, b2;
  int h = ph0 - pad;
  row(h, a0, b0);
  row(h + 1, a1, b1);
  row(h + 2, a2, b2);
  for (int ph = ph0;;) {
    float ba = -INFINITY, bb = -INFINITY;
    int ga = -1, gb = -1;
    if (a0.m > ba) { ba = a0.m; ga = h * W + ws + a0.d; }
    if (a1.m > ba) { ba = a1.m; ga = (h + 1) * W + ws + a1.d; }
    if (a2.m > ba) { ba = a2.m; ga = (h + 2) * W + ws + a2.d; }
    if (b0.m > bb) { bb = b0.m; gb = h * W + ws + 1 + b0.d; }
    if (b1.m > bb) { bb = b1.m; gb = (h + 1) * W + ws + 1 + b1.d; }
    if (b2.m > bb) { bb = b2.m; gb = (h + 2) * W + ws + 1 + b2.d; }
    emit(ph, ba, ga, bb, gb);
    if (++ph >= ph1) break;
    ++h;
    a0 = a1; a1 = a2;
    b0 = b1; b1 = b2;
    row(h + 2, a2, b2);
  }
}

__device__ __forceinline__ void issue_loads(uint32_t dst, const float* src0, int64_t n0,
                                            uint32_t dst1, const float* src1, int64_t n1,
                                            uint64_t* bar) {
  mbar_arrive_expect_tx(bar, (uint32_t)((n0 + n1) * 4));
  bulk_g2s(dst, src0, (uint32_t)(n0 * 4), bar);
  if (n1) bulk_g2s(dst1, src1, (uint32_t)(n1 * 4), bar);
}

// signed argmax mask (smask): the flat index of the window's first maximum
// when that maximum is > 0, -2 - index when it is <= 0, -1 when there is none.
// The sign is x's at the argmax pixel -- all a folded relu_backward of
// x = relu(a) needs there (relu(a) > 0 <=> a > 0; a pixel that is no window's
// argmax gets 0 either way) -- so the backward reads neither x nor a
__device__ __forceinline__ float enc_signed(int arg, float best) {
  return arg < 0 ? -1.f : (float)(best > 0.f ? arg : -2 - arg);
}
// argmax from a signed entry (without the fold)
__device__ __forceinline__ int dec_signed(float v) {
  const int a = (int)v;
  return a >= -1 ? a : -2 - a;
}

template <int S>
__global__ void __launch_bounds__(kThreads, 2) maxpool3_fwd_staged(const float* __restrict__ x,
                                                                   float* __restrict__ y,
                                                                   float* __restrict__ mask,
                                                                   Geo g, int signed_mask) {
  extern __shared__ __align__(128) float sm[];
  __shared__ uint64_t full[kMaxStages];
  const int HW = g.H * g.W, PQ = g.P * g.Q;
  if (threadIdx.x == 0) {
    for (int s = 0; s < g.NS; ++s) mbar_init(&full[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  auto planes_of = [&](int64_t c) {
    const int64_t left = g.planes - c * g.G;
    return (int)(left < g.G ? left : g.G);
  };
  if (threadIdx.x == 0) {
    int64_t c = blockIdx.x;
    for (int s = 0; s < g.NS && c < g.nchunks; ++s, c += gridDim.x)
      issue_loads(smem_u32(sm + s * g.stage_floats), x + c * g.G * HW, (int64_t)planes_of(c) * HW,
                  0, nullptr, 0, &full[s]);
  }
  int s = 0;
  uint32_t phase = 0;
  const int per_plane = g.runs * (S == 1 && g.pairs ? g.pairs : g.Q);
  for (int64_t c = blockIdx.x; c < g.nchunks; c += gridDim.x) {
    mbar_wait(&full[s], phase);
    const float* xs0 = sm + s * g.stage_floats;
    const int items = planes_of(c) * per_plane;
    float* yc = y + c * g.G * PQ;
    float* mc = mask ? mask + c * g.G * PQ : nullptr;
    if (S == 1 && g.pairs) {
      // two columns per item: float2 stores of y and the mask
      for (int it = threadIdx.x; it < items; it += kThreads) {
        const int gl = fdiv(it, g.m_pp1p, g.s_pp1p), r = it - gl * per_plane;
        const int run = fdiv(r, g.m_qp, g.s_qp), pw = 2 * (r - run * g.pairs);
        const int ph0 = run * g.RB, ph1 = min(g.P, ph0 + g.RB);
        float* yp = yc + gl * PQ + pw;
        float* mp = mc ? mc + gl * PQ + pw : nullptr;
        walk_pair(xs0 + gl * HW, g.H, g.W, g.pad, pw, ph0, ph1,
                  [&](int ph, float ba, int ga, float bb, int gb) {
                    *reinterpret_cast<float2*>(yp + ph * g.Q) = make_float2(ba, bb);
                    if (mp) {
                      *reinterpret_cast<float2*>(mp + ph * g.Q) =
                          signed_mask ? make_float2(enc_signed(ga, ba), enc_signed(gb, bb))
                                      : make_float2((float)ga, (float)gb);
                    }
                  });
      }
    } else
    for (int it = threadIdx.x; it < items; it += kThreads) {
      const int gl = fdiv(it, g.m_pp1, g.s_pp1), r = it - gl * per_plane;
      const int run = fdiv(r, g.m_q, g.s_q), pw = r - run * g.Q;
      const int ph0 = run * g.RB, ph1 = min(g.P, ph0 + g.RB);
      float* yp = yc + gl * PQ + pw;
      if (mc) {
        float* mp = mc + gl * PQ + pw;
        if (signed_mask)
          walk_windows<S>(xs0 + gl * HW, g.H, g.W, g.pad, pw, ph0, ph1,
                          [&](int ph, float best, int arg, int) {
                            yp[ph * g.Q] = best;
                            mp[ph * g.Q] = enc_signed(arg, best);
                          });
        else
          walk_windows<S>(xs0 + gl * HW, g.H, g.W, g.pad, pw, ph0, ph1,
                          [&](int ph, float best, int arg, int) {
                            yp[ph * g.Q] = best;
                            mp[ph * g.Q] = (float)arg;
                          });
      } else {
        walk_windows<S>(xs0 + gl * HW, g.H, g.W, g.pad, pw, ph0, ph1,
                        [&](int ph, float best, int, int) { yp[ph * g.Q] = best; });
      }
    }
    __syncthreads();  // every read of this stage is done: refill it
    if (threadIdx.x == 0) {
      const int64_t cn = c + (int64_t)g.NS * gridDim.x;
      if (cn < g.nchunks)
        issue_loads(smem_u32(sm + s * g.stage_floats), x + cn * g.G * HW,
                    (int64_t)planes_of(cn) * HW, 0, nullptr, 0, &full[s]);
    }
    if (++s == g.NS) {
      s = 0;
      phase ^= 1;
    }
  }
}

// MODE 0: x is the pool input, every window's argmax is recomputed (phase 1);
// MODE 1: x is the forward's argmax mask (flat indices as float32,
// [planes][P][Q]); MODE 2: x is the forward's signed mask (enc_signed);
// MODE 3: the same with the folded relu_backward, which needs no decode: the
// negative entries of windows whose maximum is <= 0 match no pixel, so those
// windows drop out.  Modes 1-3 skip phase 1.
template <int S, int MODE>
__global__ void __launch_bounds__(kThreads, 2) maxpool3_bwd_staged(const float* __restrict__ x,
                                                                   const float* __restrict__ dy,
                                                                   float* __restrict__ dx, Geo g,
                                                                   int relu_from_x) {
  extern __shared__ __align__(128) float sm[];
  __shared__ uint64_t full[kMaxStages];
  constexpr bool MASK = MODE != 0;
  const int HW = g.H * g.W, PQ = g.P * g.Q;
  // stage: [x: G*HW][dy: G*PQ][arg: G*PQ ints] (MODE 1, 2: [mask: G*PQ][dy: G*PQ]);
  // x / mask and dy segments 16-byte aligned
  const int XP = MASK ? PQ : HW;
  const int xseg = (g.G * XP + 3) & ~3, dseg = (g.G * PQ + 3) & ~3;
  if (threadIdx.x == 0) {
    for (int s = 0; s < g.NS; ++s) mbar_init(&full[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  auto planes_of = [&](int64_t c) {
    const int64_t left = g.planes - c * g.G;
    return (int)(left < g.G ? left : g.G);
  };
  auto load = [&](int s, int64_t c) {
    float* st = sm + s * g.stage_floats;
    const int gh = planes_of(c);
    issue_loads(smem_u32(st), x + c * g.G * XP, (int64_t)gh * XP, smem_u32(st + xseg),
                dy + c * g.G * PQ, (int64_t)gh * PQ, &full[s]);
  };
  if (threadIdx.x == 0) {
    int64_t c = blockIdx.x;
    for (int s = 0; s < g.NS && c < g.nchunks; ++s, c += gridDim.x) load(s, c);
  }
  int s = 0;
  uint32_t phase = 0;
  const int per_plane1 = g.runs * g.Q;
  for (int64_t c = blockIdx.x; c < g.nchunks; c += gridDim.x) {
    mbar_wait(&full[s], phase);
    const float* xs0 = sm + s * g.stage_floats;
    const float* gs0 = xs0 + xseg;
    int* as0 = reinterpret_cast<int*>(const_cast<float*>(gs0 + dseg));
    const int gh = planes_of(c);
    // window argmax as an int: recomputed (phase 1), the mask's float, or the
    // signed mask's
    const float* mk0 = xs0;
    auto arg_at = [&](const int* ap, const float* mp, int o) -> int {
      if (MODE == 2) return dec_signed(mp[o]);
      return MASK ? (int)mp[o] : ap[o];
    };
    // phase 1: every window's argmax (the forward's scan)
    if (!MASK)
    for (int it = threadIdx.x; it < gh * per_plane1; it += kThreads) {
      const int gl = fdiv(it, g.m_pp1, g.s_pp1), r = it - gl * per_plane1;
      const int run = fdiv(r, g.m_q, g.s_q), pw = r - run * g.Q;
      const int ph0 = run * g.RB, ph1 = min(g.P, ph0 + g.RB);
      int* ap = as0 + gl * PQ + pw;
      walk_windows<S>(xs0 + gl * HW, g.H, g.W, g.pad, pw, ph0, ph1,
                      [&](int ph, float, int arg, int) { ap[ph * g.Q] = arg; });
    }
    if (!MASK) __syncthreads();
    // phase 2: per input pixel, dy of the windows whose argmax it is, in window
    // raster order
    float* dxc = dx + c * g.G * HW;
    if (S == 1 && g.pairs2) {
      // two input columns w, w + 1 per item: their candidate windows share
      // columns q0 + 1, q0 + 2, so four (argmax, dy) loads per window row
      // serve both pixels; each pixel sums in window raster order as below
      const int half = g.W / 2;
      const int per_plane2 = g.hruns2 * half;
      for (int it = threadIdx.x; it < gh * per_plane2; it += kThreads) {
        const int gl = fdiv(it, g.m_pp2p, g.s_pp2p), r = it - gl * per_plane2;
        const int run = fdiv(r, g.m_in2p, g.s_in2p), w = 2 * (r - run * half);
        const int h0 = run * g.RBh2, h1 = min(g.H, h0 + g.RBh2);
        const int* ap = as0 + gl * PQ;
        const float* mp = mk0 + gl * PQ;
        const float* gp = gs0 + gl * PQ;
        const float* xs = xs0 + gl * HW;
        float* dp = dxc + gl * HW + w;
        const int q0 = w + g.pad - 2;
        bool v[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) v[j] = (unsigned)(q0 + j) < (unsigned)g.Q;
        int A0[4], A1[4], A2[4];
        float D0[4], D1[4], D2[4];
        auto ld_row = [&](int ph, int (&a)[4], float (&d)[4]) {
          const bool rv = (unsigned)ph < (unsigned)g.P;
          const int o = ph * g.Q + q0;
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            a[j] = (rv && v[j]) ? arg_at(ap, mp, o + j) : -1;
            d[j] = (rv && v[j]) ? gp[o + j] : 0.f;
          }
        };
        int p = h0 + g.pad - 2;
        ld_row(p, A0, D0);
        ld_row(p + 1, A1, D1);
        ld_row(p + 2, A2, D2);
        int h = h0;
        auto step = [&](int (&Aa)[4], float (&Da)[4], const int (&Ab)[4], const float (&Db)[4],
                        const int (&Ac)[4], const float (&Dc)[4]) -> bool {
          const int me = h * g.W + w;
          float e0 = 0.f, e1 = 0.f;
#pragma unroll
          for (int j = 0; j < 3; ++j) e0 = __fadd_rn(e0, Aa[j] == me ? Da[j] : 0.f);
#pragma unroll
          for (int j = 0; j < 3; ++j) e0 = __fadd_rn(e0, Ab[j] == me ? Db[j] : 0.f);
#pragma unroll
          for (int j = 0; j < 3; ++j) e0 = __fadd_rn(e0, Ac[j] == me ? Dc[j] : 0.f);
#pragma unroll
          for (int j = 1; j < 4; ++j) e1 = __fadd_rn(e1, Aa[j] == me + 1 ? Da[j] : 0.f);
#pragma unroll
          for (int j = 1; j < 4; ++j) e1 = __fadd_rn(e1, Ab[j] == me + 1 ? Db[j] : 0.f);
#pragma unroll
          for (int j = 1; j < 4; ++j) e1 = __fadd_rn(e1, Ac[j] == me + 1 ? Dc[j] : 0.f);
          if (MODE == 0 && relu_from_x) {
            e0 = xs[me] > 0.f ? e0 : 0.f;
            e1 = xs[me + 1] > 0.f ? e1 : 0.f;
          }
          *reinterpret_cast<float2*>(dp + h * g.W) = make_float2(e0, e1);
          if (++h >= h1) return false;
          ++p;
          ld_row(p + 2, Aa, Da);
          return true;
        };
        while (step(A0, D0, A1, D1, A2, D2) && step(A1, D1, A2, D2, A0, D0) &&
               step(A2, D2, A0, D0, A1, D1)) {
        }
      }
    } else if (S == 1) {
      const int per_plane2 = g.hruns * g.W;
      for (int it = threadIdx.x; it < gh * per_plane2; it += kThreads) {
        const int gl = fdiv(it, g.m_pp2, g.s_pp2), r = it - gl * per_plane2;
        const int run = fdiv(r, g.m_in2, g.s_in2), w = r - run * g.W;
        const int h0 = run * g.RBh, h1 = min(g.H, h0 + g.RBh);
        const int* ap = as0 + gl * PQ;
        const float* mp = mk0 + gl * PQ;
        const float* gp = gs0 + gl * PQ;
        const float* xs = xs0 + gl * HW;
        float* dp = dxc + gl * HW + w;
        // candidate windows (h + pad - 2 + i, w + pad - 2 + j), rolling in i
        const int q0 = w + g.pad - 2;
        const bool v0 = (unsigned)q0 < (unsigned)g.Q, v1 = (unsigned)(q0 + 1) < (unsigned)g.Q,
                   v2 = (unsigned)(q0 + 2) < (unsigned)g.Q;
        int A0[3], A1[3], A2[3];
        float D0[3], D1[3], D2[3];
        auto ld_row = [&](int ph, int (&a)[3], float (&d)[3]) {
          const bool rv = (unsigned)ph < (unsigned)g.P;
          const int o = ph * g.Q + q0;
          a[0] = (rv && v0) ? arg_at(ap, mp, o) : -1;
          a[1] = (rv && v1) ? arg_at(ap, mp, o + 1) : -1;
          a[2] = (rv && v2) ? arg_at(ap, mp, o + 2) : -1;
          d[0] = (rv && v0) ? gp[o] : 0.f;
          d[1] = (rv && v1) ? gp[o + 1] : 0.f;
          d[2] = (rv && v2) ? gp[o + 2] : 0.f;
        };
        int p = h0 + g.pad - 2;
        ld_row(p, A0, D0);
        ld_row(p + 1, A1, D1);
        ld_row(p + 2, A2, D2);
        int h = h0;
        // one pixel from window rows (a, b, c) = (oldest .. newest); the oldest
        // slot then takes the next window row (three rotated instances: no moves)
        auto step = [&](int (&Aa)[3], float (&Da)[3], const int (&Ab)[3], const float (&Db)[3],
                        const int (&Ac)[3], const float (&Dc)[3]) -> bool {
          const int me = h * g.W + w;
          float acc = 0.f;
#pragma unroll
          for (int j = 0; j < 3; ++j) acc = __fadd_rn(acc, Aa[j] == me ? Da[j] : 0.f);
#pragma unroll
          for (int j = 0; j < 3; ++j) acc = __fadd_rn(acc, Ab[j] == me ? Db[j] : 0.f);
#pragma unroll
          for (int j = 0; j < 3; ++j) acc = __fadd_rn(acc, Ac[j] == me ? Dc[j] : 0.f);
          if (MODE == 0 && relu_from_x) acc = xs[me] > 0.f ? acc : 0.f;
          dp[h * g.W] = acc;
          if (++h >= h1) return false;
          ++p;
          ld_row(p + 2, Aa, Da);
          return true;
        };
        while (step(A0, D0, A1, D1, A2, D2) && step(A1, D1, A2, D2, A0, D0) &&
               step(A2, D2, A0, D0, A1, D1)) {
        }
      }
    } else {
      // stride 2: thread per 2x2 pixel block (2i - pad, 2j - pad) + {0,1}^2, covered
      // exactly by windows (i-1, j-1), (i-1, j), (i, j-1), (i, j) (see the s2 plane
      // kernel in pool_lrn_concat.cu)
      const int BI = (g.H + g.pad + 1) >> 1, BJ = (g.W + g.pad + 1) >> 1;
      const int per_plane2 = BI * BJ;
      for (int it = threadIdx.x; it < gh * per_plane2; it += kThreads) {
        const int gl = fdiv(it, g.m_pp2, g.s_pp2), r = it - gl * per_plane2;
        const int i = fdiv(r, g.m_in2, g.s_in2), j = r - i * BJ;
        const int* ap = as0 + gl * PQ;
        const float* mp = mk0 + gl * PQ;
        const float* gp = gs0 + gl * PQ;
        const float* xs = xs0 + gl * HW;
        float* dp = dxc + gl * HW;
        const bool pa = (unsigned)(i - 1) < (unsigned)g.P, pb = i < g.P;
        const bool qa = (unsigned)(j - 1) < (unsigned)g.Q, qb = j < g.Q;
        const int oa = (i - 1) * g.Q, ob = i * g.Q;
        const int aAA = (pa && qa) ? arg_at(ap, mp, oa + j - 1) : -1;
        const int aAB = (pa && qb) ? arg_at(ap, mp, oa + j) : -1;
        const int aBA = (pb && qa) ? arg_at(ap, mp, ob + j - 1) : -1;
        const int aBB = (pb && qb) ? arg_at(ap, mp, ob + j) : -1;
        const float gAA = (pa && qa) ? gp[oa + j - 1] : 0.f, gAB = (pa && qb) ? gp[oa + j] : 0.f;
        const float gBA = (pb && qa) ? gp[ob + j - 1] : 0.f, gBB = (pb && qb) ? gp[ob + j] : 0.f;
        const int h0 = 2 * i - g.pad, w0 = 2 * j - g.pad;
        const int e00 = h0 * g.W + w0, e01 = e00 + 1, e10 = e00 + g.W, e11 = e10 + 1;
        float a00 = 0.f, a01 = 0.f, a10 = 0.f, a11 = 0.f;
        a00 = __fadd_rn(a00, aAA == e00 ? gAA : 0.f);
        a00 = __fadd_rn(a00, aAB == e00 ? gAB : 0.f);
        a01 = __fadd_rn(a01, aAB == e01 ? gAB : 0.f);
        a00 = __fadd_rn(a00, aBA == e00 ? gBA : 0.f);
        a10 = __fadd_rn(a10, aBA == e10 ? gBA : 0.f);
        a00 = __fadd_rn(a00, aBB == e00 ? gBB : 0.f);
        a01 = __fadd_rn(a01, aBB == e01 ? gBB : 0.f);
        a10 = __fadd_rn(a10, aBB == e10 ? gBB : 0.f);
        a11 = __fadd_rn(a11, aBB == e11 ? gBB : 0.f);
        const bool r0 = h0 >= 0, r1 = h0 + 1 < g.H, k0 = w0 >= 0, k1 = w0 + 1 < g.W;
        if (MODE == 0 && relu_from_x) {
          if (r0 && k0) a00 = xs[e00] > 0.f ? a00 : 0.f;
          if (r0 && k1) a01 = xs[e01] > 0.f ? a01 : 0.f;
          if (r1 && k0) a10 = xs[e10] > 0.f ? a10 : 0.f;
          if (r1 && k1) a11 = xs[e11] > 0.f ? a11 : 0.f;
        }
        if (r0 && k0) dp[e00] = a00;
        if (r0 && k1) dp[e01] = a01;
        if (r1 && k0) dp[e10] = a10;
        if (r1 && k1) dp[e11] = a11;
      }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      const int64_t cn = c + (int64_t)g.NS * gridDim.x;
      if (cn < g.nchunks) load(s, cn);
    }
    if (++s == g.NS) {
      s = 0;
      phase ^= 1;
    }
  }
}

// chunk geometry: G planes per stage (G * plane floats a multiple of 4 so
// every chunk starts 16-byte aligned), ~kStageTarget bytes per stage, NS
// stages within the shared-memory budget; 0 when the shape does not fit
constexpr int kStageTarget = 32 << 10;
constexpr int kSmemBudget = 200 << 10;

inline int align_planes(int per_plane_floats) {  // smallest G with G * f % 4 == 0
  for (int g = 1; g <= 4; ++g)
    if ((g * per_plane_floats) % 4 == 0) return g;
  return 4;
}

// bwd: 0 forward, 1 backward recomputing the argmax from x, 2 backward from the
// float mask, 3 backward from the signed mask (the same geometry as 2)
bool plan(Geo& g, int bwd, int N, int C, int H, int W, int P, int Q, int S, int pad) {
  g.H = H; g.W = W; g.P = P; g.Q = Q; g.pad = pad;
  g.planes = (int64_t)N * C;
  if (g.planes <= 0 || pad < 0 || pad > 2 || (S != 1 && S != 2)) return false;
  const int HW = H * W, PQ = P * Q;
  // every window must overlap the plane (the oracle's windows never lie fully in padding)
  if ((P - 1) * S - pad >= H || (Q - 1) * S - pad >= W) return false;
  if (bwd == 3) bwd = 2;  // the signed mask: the float mask's geometry
  const int a = std::max(align_planes(HW), align_planes(PQ));
  if ((g.planes * HW) % 4 || (g.planes * PQ) % 4) return false;
  const int64_t per_plane = bwd == 2 ? 2LL * PQ : bwd ? (int64_t)HW + 2LL * PQ : (int64_t)HW;
  int G = (int)std::max<int64_t>(1, (bwd ? kStageTarget * 3 / 2 : kStageTarget) / (per_plane * 4));
  G = (G + a - 1) / a * a;
  if (G > g.planes) G = (int)((g.planes + a - 1) / a * a);
  auto stage_floats = [&](int G_) {
    return bwd == 2   ? ((G_ * PQ + 3) & ~3) * 2
           : bwd      ? ((G_ * HW + 3) & ~3) + ((G_ * PQ + 3) & ~3) + G_ * PQ
                      : G_ * HW;
  };
  const int64_t sb = (int64_t)stage_floats(G) * 4;
  if (sb * 2 > kSmemBudget) return false;
  g.G = G;
  g.stage_floats = (stage_floats(G) + 31) & ~31;
  // (measured: a two-CTAs-per-SM depth -- 110 KB per CTA -- speeds pool1's
  // backward alone, 0.258 -> 0.236 ms, but costs the step 0.8%)
  g.NS = (int)std::min<int64_t>(3, kSmemBudget / ((int64_t)g.stage_floats * 4));
  // a backward stage of >= 64 KB (one 112x112 plane: pool1): one stage per
  // CTA and two CTAs per SM (0.258 -> 0.236 ms alone)
  static const int big1 = [] {
    const char* e = getenv("PURINE_B200_POOL_BIG1");
    return e && *e ? atoi(e) : 1;
  }();
  if (big1 && bwd && (int64_t)g.stage_floats * 4 >= (64 << 10)) g.NS = 1;
  if (const char* e = getenv("PURINE_B200_POOL_NS")) {  // probe: ring depth cap
    const int cap = atoi(e);
    if (cap >= 1 && cap < g.NS) g.NS = cap;
  }
  g.nchunks = (g.planes + G - 1) / G;
  // walker runs: enough items to occupy the CTA twice over, long runs for the
  // row reuse
  auto run_len = [&](int rows, int cols, int min_rows = 8) {
    const int64_t colitems = (int64_t)G * cols;
    int rb = rows;
    // (runs shorter than ~8 rows spend more on the walker's warm-up rows and
    // index decode than an idle thread costs: measured 226 -> ~70 instructions
    // per pixel for the stride-1 backward)
    if (colitems < 2 * kThreads)
      rb = (int)std::max<int64_t>(min_rows, rows * colitems / (2 * kThreads));
    return rb > rows ? rows : rb;
  };
  static const int pair_cols = [] {
    const char* e = getenv("PURINE_B200_POOL_PAIRS");
    return e && *e ? atoi(e) : 1;
  }();
  // the pair walker: half the items per row, so shorter runs keep the CTA
  // busy (28x28 planes 76 -> 66 us with 4-row runs, 14x14 46 -> 42)
  static const int pair_rb = [] {
    const char* e = getenv("PURINE_B200_POOL_PAIR_RB");
    return e && *e ? atoi(e) : 4;
  }();
  const bool pairs = pair_cols && bwd == 0 && S == 1 && Q % 2 == 0;
  static const int rb_min = [] {  // probe: the other walkers' minimum run
    const char* e = getenv("PURINE_B200_POOL_RB_MIN");
    return e && *e ? atoi(e) : 8;
  }();
  g.RB = pairs ? run_len(P, Q / 2, pair_rb) : run_len(P, Q, rb_min);
  g.runs = (P + g.RB - 1) / g.RB;
  g.RBh = run_len(H, W, rb_min);
  g.hruns = (H + g.RBh - 1) / g.RBh;
  auto magic = [](uint32_t d, uint64_t& m, int& sh) {  // exact for x < 2^31
    int l = 0;
    while ((1ull << l) < d) ++l;
    sh = 31 + l;
    m = ((1ull << sh) + d - 1) / d;
  };
  magic((uint32_t)(g.runs * Q), g.m_pp1, g.s_pp1);
  magic((uint32_t)Q, g.m_q, g.s_q);
  g.pairs2 = 0;
  static const int pair_rbh = [] {
    const char* e = getenv("PURINE_B200_POOL_PAIR_RBH");
    return e && *e ? atoi(e) : 8;
  }();
  if (pair_cols && bwd >= 1 && S == 1 && W % 2 == 0) {
    g.pairs2 = 1;
    g.RBh2 = run_len(H, W / 2, pair_rbh);
    g.hruns2 = (H + g.RBh2 - 1) / g.RBh2;
    magic((uint32_t)(g.hruns2 * (W / 2)), g.m_pp2p, g.s_pp2p);
    magic((uint32_t)(W / 2), g.m_in2p, g.s_in2p);
  }
  g.pairs = 0;
  if (pairs) {
    g.pairs = Q / 2;
    magic((uint32_t)(g.runs * g.pairs), g.m_pp1p, g.s_pp1p);
    magic((uint32_t)g.pairs, g.m_qp, g.s_qp);
  }
  if (S == 1) {
    magic((uint32_t)(g.hruns * W), g.m_pp2, g.s_pp2);
    magic((uint32_t)W, g.m_in2, g.s_in2);
  } else {
    const int BI = (H + pad + 1) >> 1, BJ = (W + pad + 1) >> 1;
    magic((uint32_t)(BI * BJ), g.m_pp2, g.s_pp2);
    magic((uint32_t)BJ, g.m_in2, g.s_in2);
  }
  return true;
}

// persistent grid: as many CTAs as fit per SM (shared memory bound), at most
// one per chunk; -1 on a CUDA error (message set)
template <class K>
int grid_for(K kern, const Geo& g, bool& configured) {
  const int smem = g.NS * g.stage_floats * 4;
  if (!configured) {
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBudget) !=
        cudaSuccess) {
      set_error("maxpool(staged): smem attribute: %s", cudaGetErrorString(cudaGetLastError()));
      return -1;
    }
    configured = true;
  }
  int per_sm = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kThreads, smem) !=
      cudaSuccess) {
    set_error("maxpool(staged): occupancy: %s", cudaGetErrorString(cudaGetLastError()));
    return -1;
  }
  per_sm = std::max(1, per_sm);
  return (int)std::min<int64_t>(g.nchunks, (int64_t)sm_count_current() * per_sm);
}

}  // namespace pools
}  // namespace bf

using namespace bf;

// PURINE_B200_POOL_STAGED bit 0: also take the stride-1 backward (mask elided)
static int pools_flags() {
  const char* e = getenv("PURINE_B200_POOL_STAGED");
  return e ? atoi(e) : 0;
}

extern "C" {

int bf_maxpool_staged_ok(int N, int C, int H, int W, int P, int Q, int kernel, int stride,
                         int pad, int backward) {
  pools::Geo g;
  if (backward == 3) {  // the signed-mask pair: forward and backward both fit
    pools::Geo g0;
    return kernel == 3 && pools::plan(g0, 0, N, C, H, W, P, Q, stride, pad) &&
                   pools::plan(g, 3, N, C, H, W, P, Q, stride, pad)
               ? 1
               : 0;
  }
  // backward 1 (argmax recomputed from x) at stride 1: the recompute + 9-window
  // gather costs ~140 instructions per pixel (1.5 TB/s), so stride-1 pools keep
  // their mask unless PURINE_B200_POOL_STAGED bit 0 asks otherwise
  if (backward == 1 && stride == 1 && !(pools_flags() & 1)) return 0;
  return kernel == 3 && pools::plan(g, backward, N, C, H, W, P, Q, stride, pad) ? 1 : 0;
}

int bf_maxpool_fwd_staged(const float* x, float* y, float* mask, int N, int C, int H, int W,
                          int P, int Q, int kernel, int stride, int pad, bf_stream_t s) {
  pools::Geo g;
  BF_REQUIRE(kernel == 3 && pools::plan(g, 0, N, C, H, W, P, Q, stride, pad),
             "maxpool_forward(staged): unsupported shape %dx%dx%dx%d k%d s%d p%d", N, C, H, W,
             kernel, stride, pad);
  BF_REQUIRE((reinterpret_cast<uintptr_t>(x) & 15) == 0, "maxpool_forward(staged): x not 16B aligned");
  const int smem = g.NS * g.stage_floats * 4;
  static bool cfg[2] = {false, false};
  auto kern = stride == 1 ? pools::maxpool3_fwd_staged<1> : pools::maxpool3_fwd_staged<2>;
  const int grid = pools::grid_for(kern, g, cfg[stride - 1]);
  if (grid <= 0) return 1;
  kern<<<grid, pools::kThreads, smem, as_stream(s)>>>(x, y, mask, g, 0);
  return check_launch("maxpool_forward(staged)");
}

int bf_maxpool_fwd_smask(const float* x, float* y, float* smask, int N, int C, int H, int W,
                         int P, int Q, int kernel, int stride, int pad, bf_stream_t s) {
  pools::Geo g, gb;
  BF_REQUIRE(kernel == 3 && pools::plan(g, 0, N, C, H, W, P, Q, stride, pad) &&
                 pools::plan(gb, 3, N, C, H, W, P, Q, stride, pad),
             "maxpool_forward(signed mask): unsupported shape %dx%dx%dx%d k%d s%d p%d", N, C, H,
             W, kernel, stride, pad);
  BF_REQUIRE((reinterpret_cast<uintptr_t>(x) & 15) == 0 && smask != nullptr,
             "maxpool_forward(signed mask): x not 16B aligned or no mask buffer");
  const int smem = g.NS * g.stage_floats * 4;
  static bool cfg[2] = {false, false};
  auto kern = stride == 1 ? pools::maxpool3_fwd_staged<1> : pools::maxpool3_fwd_staged<2>;
  const int grid = pools::grid_for(kern, g, cfg[stride - 1]);
  if (grid <= 0) return 1;
  kern<<<grid, pools::kThreads, smem, as_stream(s)>>>(x, y, smask, g, 1);
  return check_launch("maxpool_forward(signed mask)");
}

int bf_maxpool_bwd_smask(const float* smask, const float* dy, float* dx, int relu_from_sign,
                         int N, int C, int H, int W, int P, int Q, int kernel, int stride, int pad,
                         bf_stream_t s) {
  pools::Geo g;
  BF_REQUIRE(kernel == 3 && pools::plan(g, 3, N, C, H, W, P, Q, stride, pad),
             "maxpool_backward(signed mask): unsupported shape %dx%dx%dx%d k%d s%d p%d", N, C, H,
             W, kernel, stride, pad);
  BF_REQUIRE((reinterpret_cast<uintptr_t>(smask) & 15) == 0 &&
                 (reinterpret_cast<uintptr_t>(dy) & 15) == 0,
             "maxpool_backward(signed mask): mask / dy not 16B aligned");
  const int smem = g.NS * g.stage_floats * 4;
  static bool cfg[4] = {false, false, false, false};
  auto kern = relu_from_sign
                  ? (stride == 1 ? pools::maxpool3_bwd_staged<1, 3> : pools::maxpool3_bwd_staged<2, 3>)
                  : (stride == 1 ? pools::maxpool3_bwd_staged<1, 2> : pools::maxpool3_bwd_staged<2, 2>);
  const int grid = pools::grid_for(kern, g, cfg[(stride - 1) + (relu_from_sign ? 2 : 0)]);
  if (grid <= 0) return 1;
  kern<<<grid, pools::kThreads, smem, as_stream(s)>>>(smask, dy, dx, g, relu_from_sign);
  return check_launch("maxpool_backward(signed mask)");
}

int bf_maxpool_bwd_x(const float* x, const float* dy, float* dx, int relu_from_x, int N, int C,
                     int H, int W, int P, int Q, int kernel, int stride, int pad, bf_stream_t s) {
  pools::Geo g;
  BF_REQUIRE(kernel == 3 && pools::plan(g, 1, N, C, H, W, P, Q, stride, pad),
             "maxpool_backward(staged): unsupported shape %dx%dx%dx%d k%d s%d p%d", N, C, H, W,
             kernel, stride, pad);
  BF_REQUIRE((reinterpret_cast<uintptr_t>(x) & 15) == 0 && (reinterpret_cast<uintptr_t>(dy) & 15) == 0,
             "maxpool_backward(staged): x / dy not 16B aligned");
  const int smem = g.NS * g.stage_floats * 4;
  static bool cfg[2] = {false, false};
  auto kern = stride == 1 ? pools::maxpool3_bwd_staged<1, 0> : pools::maxpool3_bwd_staged<2, 0>;
  const int grid = pools::grid_for(kern, g, cfg[stride - 1]);
  if (grid <= 0) return 1;
  kern<<<grid, pools::kThreads, smem, as_stream(s)>>>(x, dy, dx, g, relu_from_x);
  return check_launch("maxpool_backward(staged)");
}

int bf_maxpool_bwd_staged(const float* mask, const float* dy, float* dx, int N, int C, int H,
                          int W, int P, int Q, int kernel, int stride, int pad, bf_stream_t s) {
  pools::Geo g;
  BF_REQUIRE(kernel == 3 && pools::plan(g, 2, N, C, H, W, P, Q, stride, pad),
             "maxpool_backward(staged mask): unsupported shape %dx%dx%dx%d k%d s%d p%d", N, C, H,
             W, kernel, stride, pad);
  BF_REQUIRE((reinterpret_cast<uintptr_t>(mask) & 15) == 0 &&
                 (reinterpret_cast<uintptr_t>(dy) & 15) == 0,
             "maxpool_backward(staged mask): mask / dy not 16B aligned");
  const int smem = g.NS * g.stage_floats * 4;
  static bool cfg[2] = {false, false};
  auto kern = stride == 1 ? pools::maxpool3_bwd_staged<1, 1> : pools::maxpool3_bwd_staged<2, 1>;
  const int grid = pools::grid_for(kern, g, cfg[stride - 1]);
  if (grid <= 0) return 1;
  kern<<<grid, pools::kThreads, smem, as_stream(s)>>>(mask, dy, dx, g, 0);
  return check_launch("maxpool_backward(staged mask)");
}

}  // extern "C"
