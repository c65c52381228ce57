// Strided input convolutions (GoogLeNet conv1: 3 -> 64, 7x7 stride 2; NIN
// conv1: 11x11 stride 4) as stride-1 convolutions over a space-to-depth view.
//
// With r = S*a + i and s = S*b + j (0 <= i, j < S):
//   y[n][k][p][q] = sum_{c,r,s} w[k][c][r][s] x[n][c][S*p + r - pad][S*q + s - pad]
//                 = sum_{c',a,b} W'[k][c'][a][b] X[n][c'][p + a][q + b]
// where c' = (c*S + i)*S + j, X[n][c'][u][v] = x[n][c][S*u + i - pad][S*v + j - pad]
// (zero outside the image) and W'[k][c'][a][b] = w[k][c][S*a + i][S*b + j]
// (zero where S*a + i >= R or S*b + j >= R).  The channel count C*S^2 is
// padded to a multiple of 16 with zero channels, so the stride-1 problem
// takes engine v2's 16-channel-chunk gathers (forward) and its 16-pixel-row
// weight-gradient gathers with unit stride -- instead of the per-element
// table gather over C*R*S = 147 rows with stride-2 taps (conv1 forward at
// 87 TFLOP/s, weight gradient at 40).  The weight gradient of the view maps
// back entry by entry: dW[k][c][r][s] = dW'[k][c'][r / S][s / S].
//
// Costs: one pass writing X (1.4x the input for conv1, recomputed in the
// backward: ~30 us each), two tiny weight re-layouts, and zero taps in the
// contraction (256 vs 147 reduction rows for conv1; the weight gradient's
// two 128-row M tiles are as many as before).
#include <stdlib.h>

#include <algorithm>

#include "gemm_common.cuh"
#include "gemm_engines.cuh"

namespace bf {
namespace s2d {

struct Geo {
  int N, C, H, W, K, R, S, P, Q, pad;
  int Cs, Rs, Hs, Ws;  // view: channels (padded), taps, plane
};

inline bool make_geo(const ConvShape& g, Geo& v) {
  v = Geo{g.N, g.C, g.H, g.W, g.K, g.R, g.stride, g.P, g.Q, g.pad, 0, 0, 0, 0};
  if (g.stride < 2 || g.R != g.S || g.R <= g.stride) return false;
  const int cv = g.C * g.stride * g.stride;
  v.Cs = (cv + 15) / 16 * 16;
  if (v.Cs > 64) return false;  // wide inputs are not worth a view
  v.Rs = (g.R + g.stride - 1) / g.stride;
  v.Hs = g.P + v.Rs - 1;
  v.Ws = g.Q + v.Rs - 1;
  return true;
}

// X[n][c'][u][v]: one thread per 4 consecutive v of one (n, c', u) row
__global__ void s2d_input_kernel(const float* __restrict__ x, float* __restrict__ X, Geo v) {
  const int64_t rows = (int64_t)v.N * v.Cs * v.Hs;
  const int vq = (v.Ws + 3) / 4;
  const int64_t total = rows * vq;
  const int S = v.S, Cv = v.C * S * S;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t row = t / vq;
    const int v0 = (int)(t - row * vq) * 4;
    const int u = (int)(row % v.Hs);
    const int64_t nc = row / v.Hs;
    const int cp = (int)(nc % v.Cs);
    const int n = (int)(nc / v.Cs);
    float* dst = X + row * v.Ws;
    float val[4] = {0.f, 0.f, 0.f, 0.f};
    if (cp < Cv) {
      const int c = cp / (S * S), ij = cp - c * S * S, i = ij / S, j = ij - i * S;
      const int h = S * u + i - v.pad;
      if ((unsigned)h < (unsigned)v.H) {
        const float* src = x + (((int64_t)n * v.C + c) * v.H + h) * v.W;
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const int w = S * (v0 + e) + j - v.pad;
          if (v0 + e < v.Ws && (unsigned)w < (unsigned)v.W) val[e] = __ldg(src + w);
        }
      }
    }
#pragma unroll
    for (int e = 0; e < 4; ++e)
      if (v0 + e < v.Ws) dst[v0 + e] = val[e];
  }
}

// W'[k][c'][a][b] from w[k][c][r][s]
__global__ void s2d_weight_kernel(const float* __restrict__ w, float* __restrict__ Wv, Geo v) {
  const int per = v.Cs * v.Rs * v.Rs;
  const int64_t total = (int64_t)v.K * per;
  const int S = v.S, Cv = v.C * S * S;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int k = (int)(t / per), rem = (int)(t - (int64_t)k * per);
    const int cp = rem / (v.Rs * v.Rs), ab = rem - cp * v.Rs * v.Rs;
    const int a = ab / v.Rs, b = ab - a * v.Rs;
    float val = 0.f;
    if (cp < Cv) {
      const int c = cp / (S * S), ij = cp - c * S * S, i = ij / S, j = ij - i * S;
      const int r = S * a + i, s = S * b + j;
      if (r < v.R && s < v.R) val = w[(((int64_t)k * v.C + c) * v.R + r) * v.R + s];
    }
    Wv[t] = val;
  }
}

// dW[k][c][r][s] = dW'[k][c'][r / S][s / S]
__global__ void s2d_wgrad_extract_kernel(const float* __restrict__ dWv, float* __restrict__ dw,
                                         Geo v) {
  const int per = v.C * v.R * v.R;
  const int64_t total = (int64_t)v.K * per;
  const int S = v.S;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int k = (int)(t / per), rem = (int)(t - (int64_t)k * per);
    const int c = rem / (v.R * v.R), rs = rem - c * v.R * v.R;
    const int r = rs / v.R, s = rs - r * v.R;
    const int cp = (c * S + r % S) * S + s % S;
    dw[t] = dWv[(((int64_t)k * v.Cs + cp) * v.Rs + r / S) * v.Rs + s / S];
  }
}

inline ConvShape view_shape(const Geo& v) {
  return ConvShape{v.N, v.Cs, v.Hs, v.Ws, v.K, v.Rs, v.Rs, v.P, v.Q, 1, 0};
}

inline int64_t align_up(int64_t b) { return (b + 1023) / 1024 * 1024; }

}  // namespace s2d

// opt-in (PURINE_B200_S2D=1): measured slower for GoogLeNet conv1 at batch
// 128 (forward 0.478 vs 0.345 ms, weight gradient 0.825 vs 0.751 ms): the
// N = 64 view tiles are MMA-issue-bound, so the 74% zero taps of the forward
// cost in full, and the weight gradient's gathers were not its bottleneck
bool s2d_enabled() {
  const char* e = getenv("PURINE_B200_S2D");
  return e && *e && atoi(e) != 0;
}

// forward through the view; -1 when the shape is not taken
int s2d_conv_fwd(const ConvShape& g, const float* x, const float* w, const EpiNCHW& epi,
                 float* ws, int64_t ws_bytes, cudaStream_t st, const char* what) {
  s2d::Geo v;
  if (!s2d_enabled() || !s2d::make_geo(g, v)) return -1;
  const int64_t xb = s2d::align_up((int64_t)v.N * v.Cs * v.Hs * v.Ws * 4);
  const int64_t wb = s2d::align_up((int64_t)v.K * v.Cs * v.Rs * v.Rs * 4);
  if (!ws || ws_bytes < xb + wb + (16LL << 20)) return -1;
  float* X = ws;
  float* Wv = reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(ws) + xb);
  float* rest = reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(ws) + xb + wb);
  const int64_t items = (int64_t)v.N * v.Cs * v.Hs * ((v.Ws + 3) / 4);
  s2d::s2d_input_kernel<<<elementwise_grid(items, 256), 256, 0, st>>>(x, X, v);
  s2d::s2d_weight_kernel<<<elementwise_grid((int64_t)v.K * v.Cs * v.Rs * v.Rs, 256), 256, 0,
                           st>>>(w, Wv, v);
  if (int rc = check_launch(what, 2)) return rc;
  const ConvShape gv = s2d::view_shape(v);
  LdFwdX la{X, gv};
  LdRowK lb{Wv, (int64_t)v.Cs * v.Rs * v.Rs};
  const int rc = tc2_conv_fwd(la, lb, v.N * v.P * v.Q, v.K, v.Cs * v.Rs * v.Rs, epi, rest,
                              ws_bytes - xb - wb, st, what);
  return rc;  // -1: declined, the caller takes the direct path
}

// weight gradient (+ fused bias gradient) through the view; -1 when not taken
int s2d_conv_wgrad(const ConvShape& g, const float* x, const float* dy, float* dw, float* db,
                   bool* db_done, float* ws, int64_t ws_bytes, cudaStream_t st,
                   const char* what) {
  s2d::Geo v;
  if (db_done) *db_done = false;
  if (!s2d_enabled() || !s2d::make_geo(g, v)) return -1;
  const int64_t xb = s2d::align_up((int64_t)v.N * v.Cs * v.Hs * v.Ws * 4);
  const int64_t wb = s2d::align_up((int64_t)v.K * v.Cs * v.Rs * v.Rs * 4);
  if (!ws || ws_bytes < xb + wb + (64LL << 20)) return -1;
  float* X = ws;
  float* dWv = reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(ws) + xb);
  float* rest = reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(ws) + xb + wb);
  const int64_t items = (int64_t)v.N * v.Cs * v.Hs * ((v.Ws + 3) / 4);
  s2d::s2d_input_kernel<<<elementwise_grid(items, 256), 256, 0, st>>>(x, X, v);
  if (int rc = check_launch(what)) return rc;
  const ConvShape gv = s2d::view_shape(v);
  LdWgradX la{X, gv};
  LdWgradDY lb{dy, gv};
  const int M = v.Cs * v.Rs * v.Rs;
  EpiT epi{dWv, nullptr, (int64_t)M};
  const int rc = tc2_conv_wgrad(la, lb, M, v.K, v.N * v.P * v.Q, epi, rest, ws_bytes - xb - wb,
                                st, what, db, db_done);
  if (rc != 0) return rc;  // -1: declined, the caller takes the direct path
  s2d::s2d_wgrad_extract_kernel<<<elementwise_grid((int64_t)v.K * v.C * v.R * v.R, 256), 256, 0,
                                  st>>>(dWv, dw, v);
  return check_launch(what);
}

}  // namespace bf
