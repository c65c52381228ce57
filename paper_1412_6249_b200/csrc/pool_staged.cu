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
#include <algorithm>

#include "common.cuh"
#include "tc_ptx.cuh"

namespace bf {
namespace pools {

using namespace tcu;

constexpr int kThreads = 256;
constexpr int kMaxStages = 4;

struct Geo {
  int H, W, P, Q, pad;
  int64_t planes;
  int G;            // planes per chunk
  int64_t nchunks;
  int RB;           // output (fwd) / input (bwd) rows per walker run
  int runs;         // ceil(rows / RB)
  int NS;           // ring stages
  int stage_floats; // floats per stage (16-byte multiple)
};

__device__ __forceinline__ void row_red(const float* __restrict__ xs, int H, int W, int h, int ws,
                                        bool c0, bool c1, bool c2, float& m, int& a) {
  m = -INFINITY;
  a = -1;
  if ((unsigned)h < (unsigned)H) {
    const float* r = xs + h * W + ws;
    const int base = h * W + ws;
    if (c0) {
      const float v = r[0];
      if (v > m) { m = v; a = base; }
    }
    if (c1) {
      const float v = r[1];
      if (v > m) { m = v; a = base + 1; }
    }
    if (c2) {
      const float v = r[2];
      if (v > m) { m = v; a = base + 2; }
    }
  }
}

__device__ __forceinline__ void pick3(const float (&rm)[3], const int (&ra)[3], float& best,
                                      int& arg) {
  best = -INFINITY;
  arg = -1;
#pragma unroll
  for (int d = 0; d < 3; ++d)
    if (rm[d] > best) {
      best = rm[d];
      arg = ra[d];
    }
}

// walk output column pw of plane xs over output rows [ph0, ph1): emit(ph, best, arg)
template <int S, class Emit>
__device__ __forceinline__ void walk_windows(const float* __restrict__ xs, const Geo& g, int pw,
                                             int ph0, int ph1, const Emit& emit) {
  const int ws = pw * S - g.pad;
  const bool c0 = (unsigned)ws < (unsigned)g.W, c1 = (unsigned)(ws + 1) < (unsigned)g.W,
             c2 = (unsigned)(ws + 2) < (unsigned)g.W;
  float rm[3];
  int ra[3];
  int h = ph0 * S - g.pad;
#pragma unroll
  for (int d = 0; d < 3; ++d) row_red(xs, g.H, g.W, h + d, ws, c0, c1, c2, rm[d], ra[d]);
  for (int ph = ph0;;) {
    float best;
    int arg;
    pick3(rm, ra, best, arg);
    emit(ph, best, arg);
    if (++ph >= ph1) break;
    h += S;
    if (S == 1) {
      rm[0] = rm[1]; ra[0] = ra[1];
      rm[1] = rm[2]; ra[1] = ra[2];
      row_red(xs, g.H, g.W, h + 2, ws, c0, c1, c2, rm[2], ra[2]);
    } else {
      rm[0] = rm[2]; ra[0] = ra[2];
      row_red(xs, g.H, g.W, h + 1, ws, c0, c1, c2, rm[1], ra[1]);
      row_red(xs, g.H, g.W, h + 2, ws, c0, c1, c2, rm[2], ra[2]);
    }
  }
}

__device__ __forceinline__ void issue_loads(uint32_t dst, const float* src0, int64_t n0,
                                            uint32_t dst1, const float* src1, int64_t n1,
                                            uint64_t* bar) {
  mbar_arrive_expect_tx(bar, (uint32_t)((n0 + n1) * 4));
  bulk_g2s(dst, src0, (uint32_t)(n0 * 4), bar);
  if (n1) bulk_g2s(dst1, src1, (uint32_t)(n1 * 4), bar);
}

template <int S>
__global__ void __launch_bounds__(kThreads) maxpool3_fwd_staged(const float* __restrict__ x,
                                                                float* __restrict__ y,
                                                                float* __restrict__ mask, Geo g) {
  extern __shared__ __align__(128) float sm[];
  __shared__ uint64_t full[kMaxStages];
  const int HW = g.H * g.W, PQ = g.P * g.Q;
  if (threadIdx.x == 0) {
    for (int s = 0; s < g.NS; ++s) mbar_init(&full[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  auto planes_of = [&](int64_t c) { const int64_t left = g.planes - c * g.G; return (int)(left < g.G ? left : g.G); };
  if (threadIdx.x == 0) {
    int64_t c = blockIdx.x;
    for (int s = 0; s < g.NS && c < g.nchunks; ++s, c += gridDim.x)
      issue_loads(smem_u32(sm + s * g.stage_floats), x + c * g.G * HW, (int64_t)planes_of(c) * HW,
                  0, nullptr, 0, &full[s]);
  }
  int s = 0;
  uint32_t phase = 0;
  for (int64_t c = blockIdx.x; c < g.nchunks; c += gridDim.x) {
    mbar_wait(&full[s], phase);
    const float* xs0 = sm + s * g.stage_floats;
    const int gh = planes_of(c);
    const int items = gh * g.runs * g.Q;
    float* yc = y + c * g.G * PQ;
    float* mc = mask ? mask + c * g.G * PQ : nullptr;
    for (int it = threadIdx.x; it < items; it += kThreads) {
      const int pw = it % g.Q, t = it / g.Q;
      const int run = t % g.runs, gl = t / g.runs;
      const int ph0 = run * g.RB, ph1 = min(g.P, ph0 + g.RB);
      float* yp = yc + gl * PQ + pw;
      float* mp = mc ? mc + gl * PQ + pw : nullptr;
      walk_windows<S>(xs0 + gl * HW, g, pw, ph0, ph1, [&](int ph, float best, int arg) {
        yp[ph * g.Q] = best;
        if (mp) mp[ph * g.Q] = (float)arg;
      });
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

template <int S>
__global__ void __launch_bounds__(kThreads) maxpool3_bwd_staged(const float* __restrict__ x,
                                                                const float* __restrict__ dy,
                                                                float* __restrict__ dx, Geo g,
                                                                int relu_from_x) {
  extern __shared__ __align__(128) float sm[];
  __shared__ uint64_t full[kMaxStages];
  const int HW = g.H * g.W, PQ = g.P * g.Q;
  // stage: [x: G*HW][dy: G*PQ][arg: G*PQ ints]; x and dy segments 16-byte aligned
  const int xseg = (g.G * HW + 3) & ~3, dseg = (g.G * PQ + 3) & ~3;
  if (threadIdx.x == 0) {
    for (int s = 0; s < g.NS; ++s) mbar_init(&full[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  auto planes_of = [&](int64_t c) { const int64_t left = g.planes - c * g.G; return (int)(left < g.G ? left : g.G); };
  auto load = [&](int s, int64_t c) {
    float* st = sm + s * g.stage_floats;
    const int gh = planes_of(c);
    issue_loads(smem_u32(st), x + c * g.G * HW, (int64_t)gh * HW, smem_u32(st + xseg),
                dy + c * g.G * PQ, (int64_t)gh * PQ, &full[s]);
  };
  if (threadIdx.x == 0) {
    int64_t c = blockIdx.x;
    for (int s = 0; s < g.NS && c < g.nchunks; ++s, c += gridDim.x) load(s, c);
  }
  int s = 0;
  uint32_t phase = 0;
  const int pruns = (g.P + g.RB - 1) / g.RB;  // phase-1 runs over output rows
  for (int64_t c = blockIdx.x; c < g.nchunks; c += gridDim.x) {
    mbar_wait(&full[s], phase);
    const float* xs0 = sm + s * g.stage_floats;
    const float* gs0 = xs0 + xseg;
    int* as0 = reinterpret_cast<int*>(const_cast<float*>(gs0 + dseg));
    const int gh = planes_of(c);
    // phase 1: every window's argmax
    {
      const int items = gh * pruns * g.Q;
      for (int it = threadIdx.x; it < items; it += kThreads) {
        const int pw = it % g.Q, t = it / g.Q;
        const int run = t % pruns, gl = t / pruns;
        const int ph0 = run * g.RB, ph1 = min(g.P, ph0 + g.RB);
        int* ap = as0 + gl * PQ + pw;
        walk_windows<S>(xs0 + gl * HW, g, pw, ph0, ph1,
                        [&](int ph, float, int arg) { ap[ph * g.Q] = arg; });
      }
    }
    __syncthreads();
    // phase 2: gather per input pixel
    float* dxc = dx + c * g.G * HW;
    const int hruns = (g.H + g.RB - 1) / g.RB;
    const int items = gh * hruns * g.W;
    for (int it = threadIdx.x; it < items; it += kThreads) {
      const int w = it % g.W, t = it / g.W;
      const int run = t % hruns, gl = t / hruns;
      const int h0 = run * g.RB, h1 = min(g.H, h0 + g.RB);
      const int* ap = as0 + gl * PQ;
      const float* gp = gs0 + gl * PQ;
      const float* xs = xs0 + gl * HW;
      float* dp = dxc + gl * HW + w;
      if (S == 1) {
        // windows (h + pad - 2 + i, w + pad - 2 + j), i, j in 0..2, rolling in i
        const int q0 = w + g.pad - 2;
        bool qv[3];
#pragma unroll
        for (int j = 0; j < 3; ++j) qv[j] = (unsigned)(q0 + j) < (unsigned)g.Q;
        int A[3][3];
        float D[3][3];
        auto ld_row = [&](int ph, int (&a)[3], float (&d)[3]) {
          const bool rv = (unsigned)ph < (unsigned)g.P;
#pragma unroll
          for (int j = 0; j < 3; ++j) {
            const bool ok = rv && qv[j];
            a[j] = ok ? ap[ph * g.Q + q0 + j] : -1;
            d[j] = ok ? gp[ph * g.Q + q0 + j] : 0.f;
          }
        };
        int p = h0 + g.pad - 2;
#pragma unroll
        for (int i = 0; i < 3; ++i) ld_row(p + i, A[i], D[i]);
        for (int h = h0;;) {
          const int me = h * g.W + w;
          float acc = 0.f;
#pragma unroll
          for (int i = 0; i < 3; ++i)
#pragma unroll
            for (int j = 0; j < 3; ++j) acc = __fadd_rn(acc, A[i][j] == me ? D[i][j] : 0.f);
          if (relu_from_x) acc = xs[h * g.W + w] > 0.f ? acc : 0.f;
          dp[h * g.W] = acc;
          if (++h >= h1) break;
          ++p;
#pragma unroll
          for (int j = 0; j < 3; ++j) {
            A[0][j] = A[1][j]; D[0][j] = D[1][j];
            A[1][j] = A[2][j]; D[1][j] = D[2][j];
          }
          ld_row(p + 2, A[2], D[2]);
        }
      } else {
        // stride 2: windows ph in [ceil((h+pad-2)/2), floor((h+pad)/2)], likewise pw
        const int wp = w + g.pad;
        const int pwh = wp >> 1, pwl = (wp & 1) ? pwh : pwh - 1;
        for (int h = h0; h < h1; ++h) {
          const int hp = h + g.pad;
          const int phh = hp >> 1, phl = (hp & 1) ? phh : phh - 1;
          const int me = h * g.W + w;
          float acc = 0.f;
          for (int ph = phl; ph <= phh; ++ph) {
            if ((unsigned)ph >= (unsigned)g.P) continue;
            for (int pw = pwl; pw <= pwh; ++pw) {
              if ((unsigned)pw >= (unsigned)g.Q) continue;
              const int o = ph * g.Q + pw;
              acc = __fadd_rn(acc, ap[o] == me ? gp[o] : 0.f);
            }
          }
          if (relu_from_x) acc = xs[h * g.W + w] > 0.f ? acc : 0.f;
          dp[h * g.W] = acc;
        }
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

bool plan(Geo& g, bool bwd, int N, int C, int H, int W, int P, int Q, int S, int pad) {
  g.H = H; g.W = W; g.P = P; g.Q = Q; g.pad = pad;
  g.planes = (int64_t)N * C;
  if (g.planes <= 0 || pad < 0 || pad > 2 || (S != 1 && S != 2)) return false;
  const int HW = H * W, PQ = P * Q;
  // every window must overlap the plane (the oracle's windows never lie fully in padding)
  if ((P - 1) * S - pad >= H || (Q - 1) * S - pad >= W) return false;
  const int a = std::max(align_planes(HW), align_planes(PQ));
  if ((g.planes * HW) % 4 || (g.planes * PQ) % 4) return false;
  const int64_t per_plane = bwd ? (int64_t)HW + 2LL * PQ : (int64_t)HW;
  int G = (int)std::max<int64_t>(1, kStageTarget / (per_plane * 4));
  G = (G + a - 1) / a * a;
  if (G > g.planes) G = (int)((g.planes + a - 1) / a * a);
  auto stage_floats = [&](int G_) {
    return bwd ? ((G_ * HW + 3) & ~3) + ((G_ * PQ + 3) & ~3) + G_ * PQ : G_ * HW;
  };
  const int64_t sb = (int64_t)stage_floats(G) * 4;
  if (sb * 2 > kSmemBudget) return false;
  g.G = G;
  g.stage_floats = (stage_floats(G) + 31) & ~31;
  g.NS = (int)std::min<int64_t>(3, kSmemBudget / ((int64_t)g.stage_floats * 4));
  g.nchunks = (g.planes + G - 1) / G;
  // walker runs: enough items to occupy the CTA, long runs for the row reuse
  const int rows = bwd ? H : P;
  const int cols = bwd ? W : Q;
  const int64_t colitems = (int64_t)G * cols;
  int RB = rows;
  if (colitems < 2 * kThreads) RB = (int)std::max<int64_t>(4, rows * colitems / (2 * kThreads));
  if (RB > rows) RB = rows;
  g.RB = RB;
  g.runs = (rows + RB - 1) / RB;
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

extern "C" {

int bf_maxpool_staged_ok(int N, int C, int H, int W, int P, int Q, int kernel, int stride,
                         int pad, int backward) {
  pools::Geo g;
  return kernel == 3 && pools::plan(g, backward != 0, N, C, H, W, P, Q, stride, pad) ? 1 : 0;
}

int bf_maxpool_fwd_staged(const float* x, float* y, float* mask, int N, int C, int H, int W,
                          int P, int Q, int kernel, int stride, int pad, bf_stream_t s) {
  pools::Geo g;
  BF_REQUIRE(kernel == 3 && pools::plan(g, false, N, C, H, W, P, Q, stride, pad),
             "maxpool_forward(staged): unsupported shape %dx%dx%dx%d k%d s%d p%d", N, C, H, W,
             kernel, stride, pad);
  BF_REQUIRE((reinterpret_cast<uintptr_t>(x) & 15) == 0, "maxpool_forward(staged): x not 16B aligned");
  const int smem = g.NS * g.stage_floats * 4;
  static bool cfg[2] = {false, false};
  auto kern = stride == 1 ? pools::maxpool3_fwd_staged<1> : pools::maxpool3_fwd_staged<2>;
  const int grid = pools::grid_for(kern, g, cfg[stride - 1]);
  if (grid <= 0) return 1;
  kern<<<grid, pools::kThreads, smem, as_stream(s)>>>(x, y, mask, g);
  return check_launch("maxpool_forward(staged)");
}

int bf_maxpool_bwd_x(const float* x, const float* dy, float* dx, int relu_from_x, int N, int C,
                     int H, int W, int P, int Q, int kernel, int stride, int pad, bf_stream_t s) {
  pools::Geo g;
  BF_REQUIRE(kernel == 3 && pools::plan(g, true, N, C, H, W, P, Q, stride, pad),
             "maxpool_backward(staged): unsupported shape %dx%dx%dx%d k%d s%d p%d", N, C, H, W,
             kernel, stride, pad);
  BF_REQUIRE((reinterpret_cast<uintptr_t>(x) & 15) == 0 && (reinterpret_cast<uintptr_t>(dy) & 15) == 0,
             "maxpool_backward(staged): x / dy not 16B aligned");
  const int smem = g.NS * g.stage_floats * 4;
  static bool cfg[2] = {false, false};
  auto kern = stride == 1 ? pools::maxpool3_bwd_staged<1> : pools::maxpool3_bwd_staged<2>;
  const int grid = pools::grid_for(kern, g, cfg[stride - 1]);
  if (grid <= 0) return 1;
  kern<<<grid, pools::kThreads, smem, as_stream(s)>>>(x, dy, dx, g, relu_from_x);
  return check_launch("maxpool_backward(staged)");
}

}  // extern "C"
