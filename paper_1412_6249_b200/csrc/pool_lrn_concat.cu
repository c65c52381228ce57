// Pooling (Caffe ceil-mode max / average), LRN across channels, channel
// concat, softmax cross-entropy and bias-gradient reductions.  All HBM-bound.
//
// Backward passes of the overlapping 3x3/2 poolings are written as GATHERS
// (one thread per input element visiting the output windows that cover it in
// row-major order), so they need no atomics and reproduce the CPU oracle's
// accumulation order bit for bit (oracle/kernels.py maxpool_backward /
// avgpool_backward).
#include <algorithm>

#include "common.cuh"

namespace bf {
namespace {

constexpr int kThreads = 256;
constexpr int kPlaneSmemMax = 100 << 10;  // shared-memory plane kernels up to 100 KB

__device__ __forceinline__ void window_rows(int o, int stride, int pad, int k, int size, int& lo,
                                            int& hi) {
  int s = o * stride - pad;
  hi = min(s + k, size);
  lo = max(s, 0);
}

__global__ void maxpool_fwd_kernel(const float* __restrict__ x, float* __restrict__ y,
                                   float* __restrict__ mask, int64_t total, int H, int W, int P,
                                   int Q, int k, int stride, int pad) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    int pw = (int)(i % Q);
    int ph = (int)((i / Q) % P);
    int64_t plane = i / ((int64_t)P * Q);
    const float* xp = x + plane * (int64_t)H * W;
    int h0, h1, w0, w1;
    window_rows(ph, stride, pad, k, H, h0, h1);
    window_rows(pw, stride, pad, k, W, w0, w1);
    float best = -INFINITY;
    int arg = -1;
    for (int h = h0; h < h1; ++h)
      for (int w = w0; w < w1; ++w) {
        float v = xp[h * W + w];
        if (v > best) {
          best = v;
          arg = h * W + w;
        }
      }
    y[i] = best;
    mask[i] = (float)arg;
  }
}

// output windows [lo, hi) along one axis that contain input coordinate h
__device__ __forceinline__ void covering(int h, int stride, int pad, int k, int P, int& lo,
                                         int& hi) {
  lo = (h + pad < k) ? 0 : (h + pad - k) / stride + 1;
  hi = min((h + pad) / stride + 1, P);
}

__global__ void maxpool_bwd_kernel(const float* __restrict__ mask, const float* __restrict__ dy,
                                   float* __restrict__ dx, int64_t total, int H, int W, int P,
                                   int Q, int k, int stride, int pad) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    int w = (int)(i % W);
    int h = (int)((i / W) % H);
    int64_t plane = i / ((int64_t)H * W);
    const float* mp = mask + plane * (int64_t)P * Q;
    const float* gp = dy + plane * (int64_t)P * Q;
    int p0, p1, q0, q1;
    covering(h, stride, pad, k, P, p0, p1);
    covering(w, stride, pad, k, Q, q0, q1);
    float me = (float)(h * W + w);
    float acc = 0.f;
    for (int p = p0; p < p1; ++p)
      for (int q = q0; q < q1; ++q)
        if (mp[p * Q + q] == me) acc = __fadd_rn(acc, gp[p * Q + q]);
    dx[i] = acc;
  }
}

__device__ __forceinline__ int avg_count(int o, int stride, int pad, int k, int size) {
  int s = o * stride - pad;
  int e = min(s + k, size + pad);
  return e - s;
}

__global__ void avgpool_fwd_kernel(const float* __restrict__ x, float* __restrict__ y,
                                   int64_t total, int H, int W, int P, int Q, int k, int stride,
                                   int pad) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    int pw = (int)(i % Q);
    int ph = (int)((i / Q) % P);
    int64_t plane = i / ((int64_t)P * Q);
    const float* xp = x + plane * (int64_t)H * W;
    int h0, h1, w0, w1;
    window_rows(ph, stride, pad, k, H, h0, h1);
    window_rows(pw, stride, pad, k, W, w0, w1);
    float acc = 0.f;
    for (int h = h0; h < h1; ++h)
      for (int w = w0; w < w1; ++w) acc = __fadd_rn(acc, xp[h * W + w]);
    float cnt = (float)(avg_count(ph, stride, pad, k, H) * avg_count(pw, stride, pad, k, W));
    y[i] = __fdiv_rn(acc, cnt);
  }
}

__global__ void avgpool_bwd_kernel(const float* __restrict__ dy, float* __restrict__ dx,
                                   int64_t total, int H, int W, int P, int Q, int k, int stride,
                                   int pad) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    int w = (int)(i % W);
    int h = (int)((i / W) % H);
    int64_t plane = i / ((int64_t)H * W);
    const float* gp = dy + plane * (int64_t)P * Q;
    int p0, p1, q0, q1;
    covering(h, stride, pad, k, P, p0, p1);
    covering(w, stride, pad, k, Q, q0, q1);
    float acc = 0.f;
    for (int p = p0; p < p1; ++p) {
      int ch = avg_count(p, stride, pad, k, H);
      for (int q = q0; q < q1; ++q) {
        float cnt = (float)(ch * avg_count(q, stride, pad, k, W));
        acc = __fadd_rn(acc, __fdiv_rn(gp[p * Q + q], cnt));
      }
    }
    dx[i] = acc;
  }
}

// LRN: one thread per element; window sums in channel order, as the oracle.
__global__ void lrn_fwd_kernel(const float* __restrict__ x, float* __restrict__ y,
                               float* __restrict__ scale, int64_t total, int C, int HW, int pre,
                               int post, float a_n, float beta, float kk) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    int c = (int)((i / HW) % C);
    int64_t base = i - (int64_t)c * HW;  // element (n, 0, hw)
    int lo = max(c - pre, 0), hi = min(c + post, C - 1);
    float acc = 0.f;
    for (int cj = lo; cj <= hi; ++cj) {
      float v = x[base + (int64_t)cj * HW];
      acc = __fadd_rn(acc, __fmul_rn(v, v));
    }
    float sc = __fadd_rn(kk, __fmul_rn(a_n, acc));
    scale[i] = sc;
    y[i] = __fmul_rn(x[i], powf(sc, -beta));
  }
}

__global__ void lrn_bwd_kernel(const float* __restrict__ x, const float* __restrict__ y,
                               const float* __restrict__ scale, const float* __restrict__ dy,
                               float* __restrict__ dx, int64_t total, int C, int HW, int pre,
                               int post, float coef, float beta) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    int c = (int)((i / HW) % C);
    int64_t base = i - (int64_t)c * HW;
    int lo = max(c - post, 0), hi = min(c + pre, C - 1);
    float acc = 0.f;
    for (int cj = lo; cj <= hi; ++cj) {
      int64_t j = base + (int64_t)cj * HW;
      acc = __fadd_rn(acc, __fdiv_rn(__fmul_rn(dy[j], y[j]), scale[j]));
    }
    float a = __fmul_rn(dy[i], powf(scale[i], -beta));
    float b = __fmul_rn(__fmul_rn(coef, x[i]), acc);
    dx[i] = __fsub_rn(a, b);
  }
}

// concat: copy one part [N][Ci*HW] into / out of the stacked [N][Ctot*HW]
__global__ void concat_part_kernel(const float* __restrict__ src, float* __restrict__ dst,
                                   int64_t chunk, int64_t src_stride, int64_t dst_stride,
                                   int64_t total) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    int64_t n = i / chunk, e = i - n * chunk;
    dst[n * dst_stride + e] = src[n * src_stride + e];
  }
}

__global__ void concat_part_v4(const float4* __restrict__ src, float4* __restrict__ dst,
                               int64_t chunk, int64_t src_stride, int64_t dst_stride,
                               int64_t total) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    int64_t n = i / chunk, e = i - n * chunk;
    dst[n * dst_stride + e] = src[n * src_stride + e];
  }
}

int copy_rows(const float* src, float* dst, int64_t N, int64_t chunk, int64_t src_stride,
              int64_t dst_stride, cudaStream_t st) {
  int64_t total = N * chunk;
  if (total <= 0) return 0;
  bool v4 = chunk % 4 == 0 && src_stride % 4 == 0 && dst_stride % 4 == 0 && aligned16(src) &&
            aligned16(dst);
  if (v4)
    concat_part_v4<<<elementwise_grid(total / 4, kThreads), kThreads, 0, st>>>(
        reinterpret_cast<const float4*>(src), reinterpret_cast<float4*>(dst), chunk / 4,
        src_stride / 4, dst_stride / 4, total / 4);
  else
    concat_part_kernel<<<elementwise_grid(total, kThreads), kThreads, 0, st>>>(
        src, dst, chunk, src_stride, dst_stride, total);
  return check_launch("concat");
}

// softmax cross-entropy: one CTA per row
__device__ __forceinline__ float block_reduce(float v, float* red, bool is_max) {
  for (int o = 16; o > 0; o >>= 1) {
    float u = __shfl_xor_sync(0xffffffffu, v, o);
    v = is_max ? fmaxf(v, u) : v + u;
  }
  int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  __syncthreads();
  if (lane == 0) red[warp] = v;
  __syncthreads();
  int nw = blockDim.x >> 5;
  v = (threadIdx.x < nw) ? red[threadIdx.x] : (is_max ? -INFINITY : 0.f);
  if (warp == 0)
    for (int o = 16; o > 0; o >>= 1) {
      float u = __shfl_xor_sync(0xffffffffu, v, o);
      v = is_max ? fmaxf(v, u) : v + u;
    }
  if (threadIdx.x == 0) red[32] = v;
  __syncthreads();
  return red[32];
}

__global__ void softmax_rows_kernel(const float* __restrict__ logits,
                                    const float* __restrict__ labels, float* __restrict__ dlogits,
                                    float* __restrict__ nll, int n, int k) {
  __shared__ float red[33];
  int row = blockIdx.x;
  const float* z = logits + (int64_t)row * k;
  float* g = dlogits + (int64_t)row * k;
  float m = -INFINITY;
  for (int j = threadIdx.x; j < k; j += blockDim.x) m = fmaxf(m, z[j]);
  m = block_reduce(m, red, true);
  float s = 0.f;
  for (int j = threadIdx.x; j < k; j += blockDim.x) s += expf(z[j] - m);
  s = block_reduce(s, red, false);
  float lab = labels[row];
  int li = (int)lab;
  bool ok = (float)li == lab && li >= 0 && li < k;
  float inv_n = (float)n;
  for (int j = threadIdx.x; j < k; j += blockDim.x) {
    float p = __fdiv_rn(expf(z[j] - m), s);
    if (j == li) p = p - 1.f;
    g[j] = __fdiv_rn(p, inv_n);
  }
  if (threadIdx.x == 0) nll[row] = ok ? -((z[li] - m) - logf(s)) : NAN;  // NaN -> finite check
}

__global__ void mean_kernel(const float* __restrict__ v, float* __restrict__ out, int n) {
  __shared__ float red[33];
  float s = 0.f;
  for (int j = threadIdx.x; j < n; j += blockDim.x) s += v[j];
  s = block_reduce(s, red, false);
  if (threadIdx.x == 0) out[0] = s / (float)n;
}

// ---- shared-memory plane kernels ---------------------------------------------------
// One CTA per (n, c) plane: the plane is staged in shared memory once, so every
// input is read from HBM once although 3x3 windows overlap; the window scan and
// the accumulation order are exactly those of the per-element kernels above
// (bit-identical results).

__global__ void maxpool_fwd_plane(const float* __restrict__ x, float* __restrict__ y,
                                  float* __restrict__ mask, int H, int W, int P, int Q, int k,
                                  int stride, int pad) {
  extern __shared__ float plane[];
  const int64_t pl = blockIdx.x;
  const float* xp = x + pl * (int64_t)H * W;
  const int HW = H * W;
  for (int i = threadIdx.x; i < HW; i += blockDim.x) plane[i] = xp[i];
  __syncthreads();
  float* yp = y + pl * (int64_t)P * Q;
  float* mp = mask + pl * (int64_t)P * Q;
  for (int o = threadIdx.x; o < P * Q; o += blockDim.x) {
    int ph = o / Q, pw = o - ph * Q;
    int h0, h1, w0, w1;
    window_rows(ph, stride, pad, k, H, h0, h1);
    window_rows(pw, stride, pad, k, W, w0, w1);
    float best = -INFINITY;
    int arg = -1;
    for (int h = h0; h < h1; ++h)
      for (int w = w0; w < w1; ++w) {
        float v = plane[h * W + w];
        if (v > best) {
          best = v;
          arg = h * W + w;
        }
      }
    yp[o] = best;
    mp[o] = (float)arg;
  }
}

__global__ void maxpool_bwd_plane(const float* __restrict__ mask, const float* __restrict__ dy,
                                  float* __restrict__ dx, int H, int W, int P, int Q, int k,
                                  int stride, int pad) {
  extern __shared__ float sm[];
  float* ms = sm;
  float* gs = sm + P * Q;
  const int64_t pl = blockIdx.x;
  const int PQ = P * Q;
  for (int i = threadIdx.x; i < PQ; i += blockDim.x) {
    ms[i] = mask[pl * PQ + i];
    gs[i] = dy[pl * PQ + i];
  }
  __syncthreads();
  float* dp = dx + pl * (int64_t)H * W;
  for (int i = threadIdx.x; i < H * W; i += blockDim.x) {
    int h = i / W, w = i - h * W;
    int p0, p1, q0, q1;
    covering(h, stride, pad, k, P, p0, p1);
    covering(w, stride, pad, k, Q, q0, q1);
    float me = (float)i;
    float acc = 0.f;
    for (int p = p0; p < p1; ++p)
      for (int q = q0; q < q1; ++q)
        if (ms[p * Q + q] == me) acc = __fadd_rn(acc, gs[p * Q + q]);
    dp[i] = acc;
  }
}

// 3x3 windows (every GoogLeNet / NIN max-pool), stride S in {1, 2}: warps walk
// output rows, lanes walk output columns (no per-element division), the window
// is unrolled with clipped taps read as -inf (strict '>' never picks them).
// global -> shared staging with 4 independent 16-byte loads in flight per
// thread (the plain strided loop was latency-bound)
__device__ __forceinline__ void stage_plane(float* __restrict__ dst, const float* __restrict__ src,
                                            int n) {
  if (((reinterpret_cast<uintptr_t>(src) & 15) == 0) && (n & 3) == 0) {
    const float4* s4 = reinterpret_cast<const float4*>(src);
    float4* d4 = reinterpret_cast<float4*>(dst);
    const int n4 = n >> 2;
    for (int base = threadIdx.x; base < n4; base += 4 * blockDim.x) {
      float4 v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int i = base + u * blockDim.x;
        if (i < n4) v[u] = __ldg(s4 + i);
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int i = base + u * blockDim.x;
        if (i < n4) d4[i] = v[u];
      }
    }
  } else {
    for (int base = threadIdx.x; base < n; base += 4 * blockDim.x) {
      float v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int i = base + u * blockDim.x;
        if (i < n) v[u] = __ldg(src + i);
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int i = base + u * blockDim.x;
        if (i < n) dst[i] = v[u];
      }
    }
  }
}

// A CTA owns G consecutive (n, c) planes (G > 1 for small 14x14 / 7x7 planes);
// a warp covers 32/CW rows x CW columns so narrow rows keep the lanes busy.
template <int S, int CW>
__global__ void maxpool3_fwd_plane(const float* __restrict__ x, float* __restrict__ y,
                                   float* __restrict__ mask, int planes, int G, int H, int W,
                                   int P, int Q, int pad) {
  extern __shared__ float plane_all[];
  const int64_t pl0 = (int64_t)blockIdx.x * G;
  const int g_here = (int)(planes - pl0 < G ? planes - pl0 : G);
  const float* xp0 = x + pl0 * (int64_t)H * W;
  stage_plane(plane_all, xp0, g_here * H * W);
  __syncthreads();
  constexpr int RPW = 32 / CW;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  const int roff = lane / CW, col = lane % CW;
  for (int rr = warp * RPW + roff; rr < g_here * P; rr += nw * RPW) {
    const int g = rr / P, ph = rr - g * P;
    const float* plane = plane_all + g * H * W;
    float* yp = y + (pl0 + g) * (int64_t)P * Q;
    float* mp = mask + (pl0 + g) * (int64_t)P * Q;
    const int hs = ph * S - pad;
    for (int pw = col; pw < Q; pw += CW) {
      const int ws = pw * S - pad;
      float best = -INFINITY;
      int arg = -1;
#pragma unroll
      for (int dh = 0; dh < 3; ++dh) {
        const int h = hs + dh;
        const bool hv = (unsigned)h < (unsigned)H;
#pragma unroll
        for (int dw = 0; dw < 3; ++dw) {
          const int w = ws + dw;
          const bool ok = hv && (unsigned)w < (unsigned)W;
          const float v = ok ? plane[h * W + w] : -INFINITY;
          if (v > best) {
            best = v;
            arg = h * W + w;
          }
        }
      }
      yp[ph * Q + pw] = best;
      mp[ph * Q + pw] = (float)arg;
    }
  }
}

template <int S, int CW>
__global__ void maxpool3_bwd_plane(const float* __restrict__ mask, const float* __restrict__ dy,
                                   float* __restrict__ dx, int planes, int G, int H, int W, int P,
                                   int Q, int pad) {
  extern __shared__ float sm[];
  const int64_t pl0 = (int64_t)blockIdx.x * G;
  const int g_here = (int)(planes - pl0 < G ? planes - pl0 : G);
  const int PQ = P * Q;
  float* ms_all = sm;
  float* gs_all = sm + G * PQ;
  stage_plane(ms_all, mask + pl0 * PQ, g_here * PQ);
  stage_plane(gs_all, dy + pl0 * PQ, g_here * PQ);
  __syncthreads();
  constexpr int RPW = 32 / CW;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  const int roff = lane / CW, col = lane % CW;
  for (int rr = warp * RPW + roff; rr < g_here * H; rr += nw * RPW) {
    const int g = rr / H, h = rr - g * H;
    const float* ms = ms_all + g * PQ;
    const float* gs = gs_all + g * PQ;
    float* dp = dx + (pl0 + g) * (int64_t)H * W;
    // output rows whose window covers h: p*S - pad <= h <= p*S - pad + 2
    const int hp = h + pad;
    const int p0 = hp < 3 ? 0 : (hp - 3) / S + 1;
    const int p1 = min(hp / S + 1, P);
    for (int w = col; w < W; w += CW) {
      const int wp = w + pad;
      const int q0 = wp < 3 ? 0 : (wp - 3) / S + 1;
      const int q1 = min(wp / S + 1, Q);
      const float me = (float)(h * W + w);
      float acc = 0.f;
#pragma unroll
      for (int a = 0; a < 3; ++a) {
        const int p = p0 + a;
        if (p < p1) {
#pragma unroll
          for (int b = 0; b < 3; ++b) {
            const int q = q0 + b;
            if (q < q1 && ms[p * Q + q] == me) acc = __fadd_rn(acc, gs[p * Q + q]);
          }
        }
      }
      dp[h * W + w] = acc;
    }
  }
}

// LRN, one thread per (n, pixel) walking the channels with a 5-wide register
// window (size == 5, the GoogLeNet / AlexNet setting): each input is read once.
// Out-of-range window slots hold +0.0, which leaves the in-order sums unchanged.
__global__ void lrn5_fwd_kernel(const float* __restrict__ x, float* __restrict__ y,
                                float* __restrict__ scale, int N, int C, int HW, float a_n,
                                float beta, float kk) {
  int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= (int64_t)N * HW) return;
  int n = (int)(t / HW), hw = (int)(t - (int64_t)n * HW);
  const float* xp = x + (int64_t)n * C * HW + hw;
  float* yp = y + (int64_t)n * C * HW + hw;
  float* sp = scale + (int64_t)n * C * HW + hw;
  // window w0..w4 = sq[c-2 .. c+2]
  float w0 = 0.f, w1 = 0.f, w2, w3, w4;
  float xc = xp[0];
  w2 = __fmul_rn(xc, xc);
  float x1 = C > 1 ? xp[HW] : 0.f;
  w3 = C > 1 ? __fmul_rn(x1, x1) : 0.f;
  float x2 = C > 2 ? xp[2 * (int64_t)HW] : 0.f;
  w4 = C > 2 ? __fmul_rn(x2, x2) : 0.f;
  for (int c = 0; c < C; ++c) {
    float acc = 0.f;
    acc = __fadd_rn(acc, w0);
    acc = __fadd_rn(acc, w1);
    acc = __fadd_rn(acc, w2);
    acc = __fadd_rn(acc, w3);
    acc = __fadd_rn(acc, w4);
    float sc = __fadd_rn(kk, __fmul_rn(a_n, acc));
    sp[(int64_t)c * HW] = sc;
    yp[(int64_t)c * HW] = __fmul_rn(xc, powf(sc, -beta));
    // slide: next channel
    float xn = x1;
    x1 = x2;
    x2 = (c + 3 < C) ? xp[(int64_t)(c + 3) * HW] : 0.f;
    w0 = w1;
    w1 = w2;
    w2 = w3;
    w3 = w4;
    w4 = (c + 3 < C) ? __fmul_rn(x2, x2) : 0.f;
    xc = xn;
  }
}

__global__ void lrn5_bwd_kernel(const float* __restrict__ x, const float* __restrict__ y,
                                const float* __restrict__ scale, const float* __restrict__ dy,
                                float* __restrict__ dx, int N, int C, int HW, float coef,
                                float beta) {
  int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= (int64_t)N * HW) return;
  int n = (int)(t / HW), hw = (int)(t - (int64_t)n * HW);
  const int64_t base = (int64_t)n * C * HW + hw;
  auto ratio = [&](int c) -> float {
    int64_t j = base + (int64_t)c * HW;
    return __fdiv_rn(__fmul_rn(dy[j], y[j]), scale[j]);
  };
  float r0 = 0.f, r1 = 0.f, r2 = ratio(0);
  float r3 = C > 1 ? ratio(1) : 0.f;
  float r4 = C > 2 ? ratio(2) : 0.f;
  for (int c = 0; c < C; ++c) {
    float acc = 0.f;
    acc = __fadd_rn(acc, r0);
    acc = __fadd_rn(acc, r1);
    acc = __fadd_rn(acc, r2);
    acc = __fadd_rn(acc, r3);
    acc = __fadd_rn(acc, r4);
    int64_t i = base + (int64_t)c * HW;
    float a = __fmul_rn(dy[i], powf(scale[i], -beta));
    float b = __fmul_rn(__fmul_rn(coef, x[i]), acc);
    dx[i] = __fsub_rn(a, b);
    r0 = r1;
    r1 = r2;
    r2 = r3;
    r3 = r4;
    r4 = (c + 3 < C) ? ratio(c + 3) : 0.f;
  }
}

// bias gradient, stage 1: CTA (slice, channel) sums dy over its images and all
// pixels (fixed tree) -> partial[channel][slice]; stage 2 adds the slices in
// order.  Deterministic, and parallel over channels x image slices.
__global__ void bias_partial_kernel(const float* __restrict__ dy, float* __restrict__ part,
                                    int N, int K, int PQ, int slices) {
  __shared__ float red[33];
  const int s = blockIdx.x, c = blockIdx.y;
  const int per = (N + slices - 1) / slices;
  const int n0 = s * per, n1 = min(N, n0 + per);
  float acc = 0.f;
  if ((PQ & 3) == 0) {
    // flattened (image, float4) index space, 4 independent loads per thread
    // in flight per iteration
    const int pq4 = PQ >> 2;
    const int total = (n1 - n0) * pq4;
    const int step = blockDim.x * 4;
    for (int base = threadIdx.x; base < total; base += step) {
      float4 v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int i = base + u * blockDim.x;
        if (i < total) {
          const int n = n0 + i / pq4, e = i - (i / pq4) * pq4;
          v[u] = __ldg(reinterpret_cast<const float4*>(dy + ((int64_t)n * K + c) * PQ) + e);
        } else {
          v[u] = make_float4(0.f, 0.f, 0.f, 0.f);
        }
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) acc += (v[u].x + v[u].y) + (v[u].z + v[u].w);
    }
  } else {
    for (int n = n0; n < n1; ++n) {
      const float* row = dy + ((int64_t)n * K + c) * PQ;
      for (int e = threadIdx.x; e < PQ; e += blockDim.x) acc += row[e];
    }
  }
  acc = block_reduce(acc, red, false);
  if (threadIdx.x == 0) part[(int64_t)c * slices + s] = acc;
}

__global__ void bias_finish_kernel(const float* __restrict__ part, float* __restrict__ db, int K,
                                   int slices) {
  int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= K) return;
  float acc = 0.f;
  for (int s = 0; s < slices; ++s) acc += part[(int64_t)c * slices + s];
  db[c] = acc;
}

// per-channel sum over (n, pq): one CTA per channel, fixed tree -> deterministic
__global__ void channel_sum_kernel(const float* __restrict__ dy, float* __restrict__ db, int N,
                                   int K, int PQ) {
  __shared__ float red[33];
  int c = blockIdx.x;
  float acc = 0.f;
  int64_t total = (int64_t)N * PQ;
  for (int64_t i = threadIdx.x; i < total; i += blockDim.x) {
    int64_t n = i / PQ, e = i - n * PQ;
    acc += dy[(n * K + c) * PQ + e];
  }
  acc = block_reduce(acc, red, false);
  if (threadIdx.x == 0) db[c] = acc;
}

// column sum of [n][m]: one thread per column, rows in order
__global__ void column_sum_kernel(const float* __restrict__ dy, float* __restrict__ db, int n,
                                  int m) {
  int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= m) return;
  float acc = 0.f;
  for (int i = 0; i < n; ++i) acc += dy[(int64_t)i * m + j];
  db[j] = acc;
}

}  // namespace
}  // namespace bf

using namespace bf;

extern "C" {

int bf_maxpool_fwd(const float* x, float* y, float* mask, int N, int C, int H, int W, int P,
                   int Q, int kernel, int stride, int pad, bf_stream_t s) {
  int64_t total = (int64_t)N * C * P * Q;
  if (total <= 0) return 0;
  const int smem = H * W * 4;
  if (smem <= kPlaneSmemMax) {
    static bool attr = false;
    if (!attr) {
      BF_CUDA(cudaFuncSetAttribute(maxpool_fwd_plane, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   kPlaneSmemMax),
              "maxpool smem attribute");
      const void* fns[] = {(const void*)maxpool3_fwd_plane<1, 8>,
                           (const void*)maxpool3_fwd_plane<1, 16>,
                           (const void*)maxpool3_fwd_plane<1, 32>,
                           (const void*)maxpool3_fwd_plane<2, 8>,
                           (const void*)maxpool3_fwd_plane<2, 16>,
                           (const void*)maxpool3_fwd_plane<2, 32>};
      for (const void* f : fns)
        BF_CUDA(cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     kPlaneSmemMax),
                "maxpool smem attribute");
      attr = true;
    }
    if (kernel == 3 && (stride == 1 || stride == 2)) {
      const int planes = N * C;
      const int G = std::max(1, std::min(16, 4096 / (H * W)));
      const int blocks = (planes + G - 1) / G;
      const int sm = G * H * W * 4;
      const int cw = Q <= 8 ? 8 : (Q <= 16 ? 16 : 32);
#define BF_MP3F(SS, CC) \
  maxpool3_fwd_plane<SS, CC><<<blocks, 256, sm, as_stream(s)>>>(x, y, mask, planes, G, H, W, P, Q, pad)
      if (stride == 1) {
        if (cw == 8) BF_MP3F(1, 8); else if (cw == 16) BF_MP3F(1, 16); else BF_MP3F(1, 32);
      } else {
        if (cw == 8) BF_MP3F(2, 8); else if (cw == 16) BF_MP3F(2, 16); else BF_MP3F(2, 32);
      }
#undef BF_MP3F
      return check_launch("maxpool_forward");
    }
    maxpool_fwd_plane<<<N * C, 256, smem, as_stream(s)>>>(x, y, mask, H, W, P, Q, kernel, stride,
                                                          pad);
    return check_launch("maxpool_forward");
  }
  maxpool_fwd_kernel<<<elementwise_grid(total, kThreads), kThreads, 0, as_stream(s)>>>(
      x, y, mask, total, H, W, P, Q, kernel, stride, pad);
  return check_launch("maxpool_forward");
}

int bf_maxpool_bwd(const float* mask, const float* dy, float* dx, int N, int C, int H, int W,
                   int P, int Q, int kernel, int stride, int pad, bf_stream_t s) {
  int64_t total = (int64_t)N * C * H * W;
  if (total <= 0) return 0;
  const int smem = 2 * P * Q * 4;
  if (smem <= kPlaneSmemMax) {
    static bool attr = false;
    if (!attr) {
      BF_CUDA(cudaFuncSetAttribute(maxpool_bwd_plane, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   kPlaneSmemMax),
              "maxpool smem attribute");
      const void* fns[] = {(const void*)maxpool3_bwd_plane<1, 8>,
                           (const void*)maxpool3_bwd_plane<1, 16>,
                           (const void*)maxpool3_bwd_plane<1, 32>,
                           (const void*)maxpool3_bwd_plane<2, 8>,
                           (const void*)maxpool3_bwd_plane<2, 16>,
                           (const void*)maxpool3_bwd_plane<2, 32>};
      for (const void* f : fns)
        BF_CUDA(cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     kPlaneSmemMax),
                "maxpool smem attribute");
      attr = true;
    }
    if (kernel == 3 && (stride == 1 || stride == 2)) {
      const int planes = N * C;
      const int G = std::max(1, std::min(16, 4096 / (H * W)));
      const int blocks = (planes + G - 1) / G;
      const int sm = G * 2 * P * Q * 4;
      const int cw = W <= 8 ? 8 : (W <= 16 ? 16 : 32);
#define BF_MP3B(SS, CC) \
  maxpool3_bwd_plane<SS, CC><<<blocks, 256, sm, as_stream(s)>>>(mask, dy, dx, planes, G, H, W, P, Q, pad)
      if (stride == 1) {
        if (cw == 8) BF_MP3B(1, 8); else if (cw == 16) BF_MP3B(1, 16); else BF_MP3B(1, 32);
      } else {
        if (cw == 8) BF_MP3B(2, 8); else if (cw == 16) BF_MP3B(2, 16); else BF_MP3B(2, 32);
      }
#undef BF_MP3B
      return check_launch("maxpool_backward");
    }
    maxpool_bwd_plane<<<N * C, 256, smem, as_stream(s)>>>(mask, dy, dx, H, W, P, Q, kernel,
                                                          stride, pad);
    return check_launch("maxpool_backward");
  }
  maxpool_bwd_kernel<<<elementwise_grid(total, kThreads), kThreads, 0, as_stream(s)>>>(
      mask, dy, dx, total, H, W, P, Q, kernel, stride, pad);
  return check_launch("maxpool_backward");
}

int bf_avgpool_fwd(const float* x, float* y, int N, int C, int H, int W, int P, int Q,
                   int kernel, int stride, int pad, bf_stream_t s) {
  int64_t total = (int64_t)N * C * P * Q;
  if (total <= 0) return 0;
  avgpool_fwd_kernel<<<elementwise_grid(total, kThreads), kThreads, 0, as_stream(s)>>>(
      x, y, total, H, W, P, Q, kernel, stride, pad);
  return check_launch("avgpool_forward");
}

int bf_avgpool_bwd(const float* dy, float* dx, int N, int C, int H, int W, int P, int Q,
                   int kernel, int stride, int pad, bf_stream_t s) {
  int64_t total = (int64_t)N * C * H * W;
  if (total <= 0) return 0;
  avgpool_bwd_kernel<<<elementwise_grid(total, kThreads), kThreads, 0, as_stream(s)>>>(
      dy, dx, total, H, W, P, Q, kernel, stride, pad);
  return check_launch("avgpool_backward");
}

int bf_lrn_fwd(const float* x, float* y, float* scale, int N, int C, int H, int W, int size,
               float alpha, float beta, float k, bf_stream_t s) {
  BF_REQUIRE(size >= 1, "lrn_forward: size must be >= 1");
  int64_t total = (int64_t)N * C * H * W;
  if (total <= 0) return 0;
  int pre = (size - 1) / 2, post = size - 1 - pre;
  float a_n = alpha / (float)size;
  if (size == 5) {
    int64_t px = (int64_t)N * H * W;
    lrn5_fwd_kernel<<<(int)((px + 255) / 256), 256, 0, as_stream(s)>>>(x, y, scale, N, C, H * W,
                                                                       a_n, beta, k);
    return check_launch("lrn_forward");
  }
  lrn_fwd_kernel<<<elementwise_grid(total, kThreads), kThreads, 0, as_stream(s)>>>(
      x, y, scale, total, C, H * W, pre, post, a_n, beta, k);
  return check_launch("lrn_forward");
}

int bf_lrn_bwd(const float* x, const float* y, const float* scale, const float* dy, float* dx,
               int N, int C, int H, int W, int size, float alpha, float beta, float k,
               bf_stream_t s) {
  BF_REQUIRE(size >= 1, "lrn_backward: size must be >= 1");
  int64_t total = (int64_t)N * C * H * W;
  if (total <= 0) return 0;
  int pre = (size - 1) / 2, post = size - 1 - pre;
  float coef = 2.0f * alpha;
  coef = coef * beta;
  coef = coef / (float)size;
  if (size == 5) {
    int64_t px = (int64_t)N * H * W;
    lrn5_bwd_kernel<<<(int)((px + 255) / 256), 256, 0, as_stream(s)>>>(x, y, scale, dy, dx, N, C,
                                                                       H * W, coef, beta);
    return check_launch("lrn_backward");
  }
  lrn_bwd_kernel<<<elementwise_grid(total, kThreads), kThreads, 0, as_stream(s)>>>(
      x, y, scale, dy, dx, total, C, H * W, pre, post, coef, beta);
  (void)k;
  return check_launch("lrn_backward");
}

int bf_concat_fwd(const float* const* parts, const int* channels, int k, float* y, int N, int H,
                  int W, bf_stream_t s) {
  BF_REQUIRE(k >= 1 && k <= 32, "concat_forward: 1..32 parts");
  int64_t HW = (int64_t)H * W, Ct = 0;
  for (int i = 0; i < k; ++i) Ct += channels[i];
  int64_t off = 0;
  for (int i = 0; i < k; ++i) {
    int64_t chunk = (int64_t)channels[i] * HW;
    int rc = copy_rows(parts[i], y + off * HW, N, chunk, chunk, Ct * HW, as_stream(s));
    if (rc) return rc;
    off += channels[i];
  }
  return 0;
}

int bf_concat_bwd(const float* dy, float* const* parts, const int* channels, int k, int N, int H,
                  int W, bf_stream_t s) {
  BF_REQUIRE(k >= 1 && k <= 32, "concat_backward: 1..32 parts");
  int64_t HW = (int64_t)H * W, Ct = 0;
  for (int i = 0; i < k; ++i) Ct += channels[i];
  int64_t off = 0;
  for (int i = 0; i < k; ++i) {
    int64_t chunk = (int64_t)channels[i] * HW;
    int rc = copy_rows(dy + off * HW, parts[i], N, chunk, Ct * HW, chunk, as_stream(s));
    if (rc) return rc;
    off += channels[i];
  }
  return 0;
}

int bf_softmax_xent(const float* logits, const float* labels, float* loss, float* dlogits, int n,
                    int k, float* workspace, bf_stream_t s) {
  BF_REQUIRE(n >= 1 && k >= 1, "softmax_xent: empty logits");
  softmax_rows_kernel<<<n, 256, 0, as_stream(s)>>>(logits, labels, dlogits, workspace, n, k);
  if (int rc = check_launch("softmax_xent")) return rc;
  mean_kernel<<<1, 256, 0, as_stream(s)>>>(workspace, loss, n);
  return check_launch("softmax_xent(mean)");
}

int bf_conv2d_bwd_bias(const float* dy, float* db, int N, int K, int PQ, float* workspace,
                       int64_t ws_bytes, bf_stream_t s) {
  if (K <= 0) return 0;
  int slices = (4 * sm_count_current() + K - 1) / K;
  if (slices > N) slices = N;
  if (slices > 1 && workspace && (int64_t)K * slices * 4 <= ws_bytes) {
    bias_partial_kernel<<<dim3(slices, K), 256, 0, as_stream(s)>>>(dy, workspace, N, K, PQ,
                                                                   slices);
    if (int rc = check_launch("conv2d_backward_bias")) return rc;
    bias_finish_kernel<<<(K + 127) / 128, 128, 0, as_stream(s)>>>(workspace, db, K, slices);
    return check_launch("conv2d_backward_bias");
  }
  channel_sum_kernel<<<K, 512, 0, as_stream(s)>>>(dy, db, N, K, PQ);
  return check_launch("conv2d_backward_bias");
}

int bf_fc_bwd_bias(const float* dy, float* db, int n, int m, bf_stream_t s) {
  if (m <= 0) return 0;
  column_sum_kernel<<<(m + 127) / 128, 128, 0, as_stream(s)>>>(dy, db, n, m);
  return check_launch("fc_backward_bias");
}

}  // extern "C"
