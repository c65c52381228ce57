// Pooling (Caffe ceil-mode max / average), LRN across channels, channel
// concat, softmax cross-entropy and bias-gradient reductions.  All HBM-bound.
//
// Backward passes of the overlapping 3x3/2 poolings are written as GATHERS
// (one thread per input element visiting the output windows that cover it in
// row-major order), so they need no atomics and reproduce the CPU oracle's
// accumulation order bit for bit (oracle/kernels.py maxpool_backward /
// avgpool_backward).
#include <algorithm>
#include <cstdlib>
#include <initializer_list>

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

// relu_backward folded into the kernel producing its dy (dispatcher fusion):
// relu_g(x, g) = x > 0 ? g : 0 exactly as elementwise.cu
__device__ __forceinline__ float relu_fold(const float* __restrict__ rx, int64_t i, float v) {
  return rx ? (__ldg(rx + i) > 0.f ? v : 0.f) : v;
}

__global__ void maxpool_bwd_kernel(const float* __restrict__ mask, const float* __restrict__ dy,
                                   float* __restrict__ dx, int64_t total, int H, int W, int P,
                                   int Q, int k, int stride, int pad,
                                   const float* __restrict__ relu_x) {
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
    dx[i] = relu_fold(relu_x, i, acc);
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

// global average pooling (window = the whole plane, one output per plane):
// every input pixel gets 0 + dy / f32(H*W), the general kernel's arithmetic
// without its per-element 64-bit index divisions and window loops
__global__ void avgpool_global_bwd_kernel(const float* __restrict__ dy, float* __restrict__ dx,
                                          uint32_t total, uint32_t HW, float cnt) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += gridDim.x * blockDim.x)
    dx[i] = __fadd_rn(0.f, __fdiv_rn(__ldg(dy + i / HW), cnt));
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

// scale^-beta and a / scale for LRN.  scale >= k > 0, so the MUFU
// approximations need no special-case code: lg2/ex2.approx (~2^-22 relative)
// and rcp.approx keep y and dx within ~5e-7 relative of powf and IEEE division
// (tests hold 1e-6 on y against the oracle's numpy power).  Every LRN kernel
// uses these two, so the recomputing backward stays bit-identical to the
// explicit one.  (powf / __fdiv_rn made the LRN kernels issue-bound: ~68
// instructions per element.)
__device__ __forceinline__ float lrn_pow(float s, float nbeta) {
  float l, r;
  asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(l) : "f"(s));
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(__fmul_rn(nbeta, l)));
  return r;
}
__device__ __forceinline__ float lrn_div(float a, float s) { return __fdividef(a, s); }

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
    y[i] = __fmul_rn(x[i], lrn_pow(sc, -beta));
  }
}

__global__ void lrn_bwd_kernel(const float* __restrict__ x, const float* __restrict__ y,
                               const float* __restrict__ scale, const float* __restrict__ dy,
                               float* __restrict__ dx, int64_t total, int C, int HW, int pre,
                               int post, float coef, float beta, const float* __restrict__ relu_x) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    int c = (int)((i / HW) % C);
    int64_t base = i - (int64_t)c * HW;
    int lo = max(c - post, 0), hi = min(c + pre, C - 1);
    float acc = 0.f;
    for (int cj = lo; cj <= hi; ++cj) {
      int64_t j = base + (int64_t)cj * HW;
      acc = __fadd_rn(acc, lrn_div(__fmul_rn(dy[j], y[j]), scale[j]));
    }
    float a = __fmul_rn(dy[i], lrn_pow(scale[i], -beta));
    float b = __fmul_rn(__fmul_rn(coef, x[i]), acc);
    dx[i] = relu_fold(relu_x, i, __fsub_rn(a, b));
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
                                  int stride, int pad, const float* __restrict__ relu_x) {
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
    dp[i] = relu_fold(relu_x, pl * (int64_t)H * W + i, acc);
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

// (mask, dy) interleaved into float2 pairs while staging: one 8-byte shared
// load per candidate window in the gather below
__device__ __forceinline__ void stage_pairs(float2* __restrict__ dst, const float* __restrict__ m,
                                            const float* __restrict__ g, int n) {
  if ((((reinterpret_cast<uintptr_t>(m) | reinterpret_cast<uintptr_t>(g)) & 15) == 0) &&
      (n & 3) == 0) {
    const float4* m4 = reinterpret_cast<const float4*>(m);
    const float4* g4 = reinterpret_cast<const float4*>(g);
    float4* d4 = reinterpret_cast<float4*>(dst);
    const int n4 = n >> 2;
    for (int base = threadIdx.x; base < n4; base += 2 * blockDim.x) {
      float4 mv[2], gv[2];
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const int i = base + u * blockDim.x;
        if (i < n4) {
          mv[u] = __ldg(m4 + i);
          gv[u] = __ldg(g4 + i);
        }
      }
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const int i = base + u * blockDim.x;
        if (i < n4) {
          d4[2 * i] = make_float4(mv[u].x, gv[u].x, mv[u].y, gv[u].y);
          d4[2 * i + 1] = make_float4(mv[u].z, gv[u].z, mv[u].w, gv[u].w);
        }
      }
    }
  } else {
    for (int i = threadIdx.x; i < n; i += blockDim.x) dst[i] = make_float2(__ldg(m + i), __ldg(g + i));
  }
}

// Gather form (bit-exact with the oracle's raster-order scatter): pixel (h, w)
// sums, in window raster order, dy of the windows whose argmax it is.  At most
// ceil(3/S) windows cover it per axis; every candidate is evaluated branch-free
// (clamped index, select of +0.0: acc starts at +0.0 and can never become
// -0.0, so adding +0.0 is the identity).
template <int S, int CW>
__global__ void maxpool3_bwd_plane(const float* __restrict__ mask, const float* __restrict__ dy,
                                   float* __restrict__ dx, int planes, int G, int H, int W, int P,
                                   int Q, int pad, const float* __restrict__ relu_x) {
  extern __shared__ float2 pairs_all[];
  const int64_t pl0 = (int64_t)blockIdx.x * G;
  const int g_here = (int)(planes - pl0 < G ? planes - pl0 : G);
  const int PQ = P * Q;
  stage_pairs(pairs_all, mask + pl0 * PQ, dy + pl0 * PQ, g_here * PQ);
  __syncthreads();
  constexpr int RPW = 32 / CW;
  constexpr int NA = (3 + S - 1) / S;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  const int roff = lane / CW, col = lane % CW;
  for (int rr = warp * RPW + roff; rr < g_here * H; rr += nw * RPW) {
    const int g = rr / H, h = rr - g * H;
    const float2* pr = pairs_all + g * PQ;
    const int64_t row0 = (pl0 + g) * (int64_t)H * W + h * W;
    float* dp = dx + row0;
    // output rows whose window covers h: p*S - pad <= h <= p*S - pad + 2
    const int hp = h + pad;
    const int p0 = hp < 3 ? 0 : (hp - 3) / S + 1;
    const int p1 = min(hp / S + 1, P);
    int prow[NA];
    bool pok[NA];
#pragma unroll
    for (int a = 0; a < NA; ++a) {
      pok[a] = p0 + a < p1;
      prow[a] = (pok[a] ? p0 + a : 0) * Q;
    }
    const int hw0 = h * W;
    for (int w = col; w < W; w += CW) {
      const int wp = w + pad;
      const int q0 = wp < 3 ? 0 : (wp - 3) / S + 1;
      const int q1 = min(wp / S + 1, Q);
      const float me = (float)(hw0 + w);
      float acc = 0.f;
#pragma unroll
      for (int a = 0; a < NA; ++a) {
#pragma unroll
        for (int b = 0; b < NA; ++b) {
          const bool ok = pok[a] && q0 + b < q1;
          const float2 mg = pr[prow[a] + (ok ? q0 + b : 0)];
          acc = __fadd_rn(acc, (ok && mg.x == me) ? mg.y : 0.f);
        }
      }
      dp[w] = relu_fold(relu_x, row0 + w, acc);
    }
  }
}

#ifndef POOL_PF
#define POOL_PF 2  // rows the column walkers load ahead of their use (measured: 1-2 best)
#endif

// Column walkers for 3x3 pooling: a thread owns one output column (forward)
// or input column (backward) of one plane and walks down its rows, keeping the
// window's per-row state in registers.  Loads go straight through L1 (the
// lanes of a warp cover consecutive columns, so neighbouring windows share
// lines) and are issued POOL_PF rows ahead of their use.  No shared memory and no
// block barriers: the plane-staging kernels above serialise load -> barrier ->
// compute inside each CTA and reached only 1.3-2 TB/s on the stride-1
// Inception pools (28x28 / 14x14 / 7x7 planes).
//
// Forward, separable argmax: each input row's 3 window columns reduce to
// (first max, its index); the window's result is the first row whose row-max
// is strictly greater than the earlier rows'.  With strict '>' from -inf in
// both passes this is exactly the first maximum in window raster order, the
// plane kernels' (and the oracle's) semantics, NaN and all -inf included.
// Each row reduction serves 3 windows (stride 1).
template <int S>
__global__ void __launch_bounds__(256) maxpool3_fwd_cols(const float* __restrict__ x,
                                                         float* __restrict__ y,
                                                         float* __restrict__ mask,
                                                         int64_t threads, int H, int W, int P,
                                                         int Q, int pad) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= threads) return;
  const int64_t pl = t / Q;
  const int pw = (int)(t - pl * Q);
  const float* __restrict__ xp = x + pl * H * W;
  float* __restrict__ yp = y + pl * P * Q + pw;
  float* __restrict__ mp = mask + pl * P * Q + pw;
  const int ws = pw * S - pad;
  bool cv[3];
#pragma unroll
  for (int d = 0; d < 3; ++d) cv[d] = (unsigned)(ws + d) < (unsigned)W;
  auto ld_row = [&](int h, float (&v)[3]) {
    const bool rv = (unsigned)h < (unsigned)H;
    const int off = h * W + ws;
#pragma unroll
    for (int d = 0; d < 3; ++d) v[d] = (rv && cv[d]) ? __ldg(xp + off + d) : -INFINITY;
  };
  auto red_row = [&](int h, const float (&v)[3], float& m, int& a) {
    m = -INFINITY;
    a = -1;
#pragma unroll
    for (int d = 0; d < 3; ++d)
      if (v[d] > m) {
        m = v[d];
        a = h * W + ws + d;
      }
  };
  int hs = -pad;
  float rm[3];
  int ra[3];
#pragma unroll
  for (int j = 0; j < 3; ++j) {
    float v[3];
    ld_row(hs + j, v);
    red_row(hs + j, v, rm[j], ra[j]);
  }
  float q[POOL_PF][S][3];  // q[k]: the rows entering at output row ph + 1 + k
#pragma unroll
  for (int k = 0; k < POOL_PF; ++k)
#pragma unroll
    for (int j = 0; j < S; ++j) ld_row(hs + 3 + k * S + j, q[k][j]);
  for (int ph = 0; ph < P; ++ph, hs += S) {
    float nq[S][3];
#pragma unroll
    for (int j = 0; j < S; ++j) ld_row(hs + 3 + POOL_PF * S + j, nq[j]);
    float best = -INFINITY;
    int arg = -1;
#pragma unroll
    for (int d = 0; d < 3; ++d)
      if (rm[d] > best) {
        best = rm[d];
        arg = ra[d];
      }
    yp[(int64_t)ph * Q] = best;
    mp[(int64_t)ph * Q] = (float)arg;
    if (S == 1) {
      rm[0] = rm[1]; ra[0] = ra[1];
      rm[1] = rm[2]; ra[1] = ra[2];
      red_row(hs + 3, q[0][0], rm[2], ra[2]);
    } else {
      rm[0] = rm[2]; ra[0] = ra[2];
      red_row(hs + 3, q[0][0], rm[1], ra[1]);
      red_row(hs + 4, q[0][S - 1], rm[2], ra[2]);
    }
#pragma unroll
    for (int k = 0; k + 1 < POOL_PF; ++k)
#pragma unroll
      for (int j = 0; j < S; ++j)
#pragma unroll
        for (int d = 0; d < 3; ++d) q[k][j][d] = q[k + 1][j][d];
#pragma unroll
    for (int j = 0; j < S; ++j)
#pragma unroll
      for (int d = 0; d < 3; ++d) q[POOL_PF - 1][j][d] = nq[j][d];
  }
}

// Stride-1 backward walker: input pixel (h, w) gathers, in window raster
// order, dy of the windows (h + pad - 2 + i, w + pad - 2 + j) whose argmax it
// is (bit-exact with the oracle's raster-order scatter, as the plane kernel);
// the 3 candidate output rows' (mask, dy) triples roll down with h.
__global__ void __launch_bounds__(256) maxpool3s1_bwd_cols(const float* __restrict__ mask,
                                                           const float* __restrict__ dy,
                                                           float* __restrict__ dx, int64_t threads,
                                                           int H, int W, int P, int Q, int pad,
                                                           const float* __restrict__ relu_x) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= threads) return;
  const int64_t pl = t / W;
  const int w = (int)(t - pl * W);
  const float* __restrict__ mp = mask + pl * P * Q;
  const float* __restrict__ gp = dy + pl * P * Q;
  const int64_t obase = pl * H * W + w;
  const int q0 = w + pad - 2;
  bool qv[3];
#pragma unroll
  for (int j = 0; j < 3; ++j) qv[j] = (unsigned)(q0 + j) < (unsigned)Q;
  auto ld_row = [&](int ph, float (&m)[3], float (&g)[3]) {
    const bool rv = (unsigned)ph < (unsigned)P;
    const int off = ph * Q + q0;
#pragma unroll
    for (int j = 0; j < 3; ++j) {
      const bool ok = rv && qv[j];
      m[j] = ok ? __ldg(mp + off + j) : -1.f;
      g[j] = ok ? __ldg(gp + off + j) : 0.f;
    }
  };
  float M[3][3], G[3][3], qm[POOL_PF][3], qg[POOL_PF][3];  // q[k]: output row h + pad + 1 + k
#pragma unroll
  for (int i = 0; i < 3; ++i) ld_row(pad - 2 + i, M[i], G[i]);
#pragma unroll
  for (int k = 0; k < POOL_PF; ++k) ld_row(pad + 1 + k, qm[k], qg[k]);
  for (int h = 0; h < H; ++h) {
    float nm[3], ng[3];
    ld_row(h + pad + 1 + POOL_PF, nm, ng);
    const float me = (float)(h * W + w);
    float acc = 0.f;
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
      for (int j = 0; j < 3; ++j) acc = __fadd_rn(acc, M[i][j] == me ? G[i][j] : 0.f);
    const int64_t o = obase + (int64_t)h * W;
    dx[o] = relu_fold(relu_x, o, acc);
#pragma unroll
    for (int j = 0; j < 3; ++j) {
      M[0][j] = M[1][j]; G[0][j] = G[1][j];
      M[1][j] = M[2][j]; G[1][j] = G[2][j];
      M[2][j] = qm[0][j]; G[2][j] = qg[0][j];
#pragma unroll
      for (int k = 0; k + 1 < POOL_PF; ++k) {
        qm[k][j] = qm[k + 1][j];
        qg[k][j] = qg[k + 1][j];
      }
      qm[POOL_PF - 1][j] = nm[j];
      qg[POOL_PF - 1][j] = ng[j];
    }
  }
}

#ifndef POOL_ROW_PF
#define POOL_ROW_PF 6  // rows the warp-row kernels load ahead of their use
#endif

// Warp-row kernels for the stride-1, pad-1 3x3 pools of planes at most 32
// wide (every Inception pool: 28, 14, 7): a warp holds floor(32 / W) planes
// side by side, one lane per column, and walks their rows.  Each lane loads
// ONE element per row (fully coalesced, no redundant L1 requests) and takes
// its neighbours' columns by warp shuffle; POOL_ROW_PF rows are in flight per
// lane.  Same separable argmax / raster-order gather as the walkers above.
__global__ void __launch_bounds__(256) maxpool3s1_fwd_rows(const float* __restrict__ x,
                                                           float* __restrict__ y,
                                                           float* __restrict__ mask,
                                                           int64_t planes, int H, int W) {
  const int lane = threadIdx.x & 31;
  const int ppw = 32 / W;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int sub = lane / W, w = lane - sub * W;
  const int64_t pl = warp * ppw + sub;
  const bool act = sub < ppw && pl < planes;
  if (warp * ppw >= planes) return;  // warp-uniform
  const int64_t base = (act ? pl : 0) * H * W + w;
  const bool has_l = w > 0, has_r = w + 1 < W;
  auto ld = [&](int h) { return (act && h < H) ? __ldg(x + base + (int64_t)h * W) : -INFINITY; };
  // row reduction of input row h from this lane's element v (first max over w-1, w, w+1)
  auto red = [&](int h, float v, float& m, int& a) {
    const float l = __shfl_up_sync(0xffffffffu, v, 1), r = __shfl_down_sync(0xffffffffu, v, 1);
    const float c0 = has_l ? l : -INFINITY, c2 = has_r ? r : -INFINITY;
    m = -INFINITY;
    a = -1;
    const int i0 = h * W + w - 1;
    if (c0 > m) { m = c0; a = i0; }
    if (v > m) { m = v; a = i0 + 1; }
    if (c2 > m) { m = c2; a = i0 + 2; }
  };
  float q[POOL_ROW_PF];  // q[k] = x row k + 1 relative to the current output row
#pragma unroll
  for (int k = 0; k < POOL_ROW_PF; ++k) q[k] = ld(1 + k);
  // rows -1 (padding), 0
  float rm[3];
  int ra[3];
  rm[0] = -INFINITY;
  ra[0] = -1;
  red(0, ld(0), rm[1], ra[1]);
  for (int h = 0; h < H; ++h) {
    const float nx = ld(h + 1 + POOL_ROW_PF);
    if (h + 1 < H) {
      red(h + 1, q[0], rm[2], ra[2]);
    } else {
      rm[2] = -INFINITY;
      ra[2] = -1;
    }
    float best = -INFINITY;
    int arg = -1;
#pragma unroll
    for (int d = 0; d < 3; ++d)
      if (rm[d] > best) {
        best = rm[d];
        arg = ra[d];
      }
    if (act) {
      y[base + (int64_t)h * W] = best;
      mask[base + (int64_t)h * W] = (float)arg;
    }
    rm[0] = rm[1]; ra[0] = ra[1];
    rm[1] = rm[2]; ra[1] = ra[2];
#pragma unroll
    for (int k = 0; k + 1 < POOL_ROW_PF; ++k) q[k] = q[k + 1];
    q[POOL_ROW_PF - 1] = nx;
  }
}

__global__ void __launch_bounds__(256) maxpool3s1_bwd_rows(const float* __restrict__ mask,
                                                           const float* __restrict__ dy,
                                                           float* __restrict__ dx, int64_t planes,
                                                           int H, int W,
                                                           const float* __restrict__ relu_x) {
  const int lane = threadIdx.x & 31;
  const int ppw = 32 / W;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int sub = lane / W, w = lane - sub * W;
  const int64_t pl = warp * ppw + sub;
  const bool act = sub < ppw && pl < planes;
  if (warp * ppw >= planes) return;  // warp-uniform
  const int64_t base = (act ? pl : 0) * H * W + w;
  const bool has_l = w > 0, has_r = w + 1 < W;
  // output row p of this column: (mask, dy), (-1, 0) outside the plane
  auto ldm = [&](int p) { return (act && p < H) ? __ldg(mask + base + (int64_t)p * W) : -1.f; };
  auto ldg_ = [&](int p) { return (act && p < H) ? __ldg(dy + base + (int64_t)p * W) : 0.f; };
  // the three candidate windows of row p seen from this lane: columns w-1, w, w+1
  auto spread = [&](float m, float g, float (&M)[3], float (&G)[3]) {
    const float ml = __shfl_up_sync(0xffffffffu, m, 1), mr = __shfl_down_sync(0xffffffffu, m, 1);
    const float gl = __shfl_up_sync(0xffffffffu, g, 1), gr = __shfl_down_sync(0xffffffffu, g, 1);
    M[0] = has_l ? ml : -1.f;  G[0] = has_l ? gl : 0.f;
    M[1] = m;                  G[1] = g;
    M[2] = has_r ? mr : -1.f;  G[2] = has_r ? gr : 0.f;
  };
  float qm[POOL_ROW_PF], qg[POOL_ROW_PF];  // output row h + 1 + k
#pragma unroll
  for (int k = 0; k < POOL_ROW_PF; ++k) {
    qm[k] = ldm(1 + k);
    qg[k] = ldg_(1 + k);
  }
  float M[3][3], G[3][3];  // candidate output rows h-1, h, h+1
#pragma unroll
  for (int j = 0; j < 3; ++j) {
    M[0][j] = -1.f;
    G[0][j] = 0.f;
  }
  spread(ldm(0), ldg_(0), M[1], G[1]);
  for (int h = 0; h < H; ++h) {
    const float nm = ldm(h + 1 + POOL_ROW_PF), ng = ldg_(h + 1 + POOL_ROW_PF);
    spread(qm[0], qg[0], M[2], G[2]);  // row h + 1 (already -1 / 0 past the plane)
    const float me = (float)(h * W + w);
    float acc = 0.f;
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
      for (int j = 0; j < 3; ++j) acc = __fadd_rn(acc, M[i][j] == me ? G[i][j] : 0.f);
    if (act) {
      const int64_t o = base + (int64_t)h * W;
      dx[o] = relu_fold(relu_x, o, acc);
    }
#pragma unroll
    for (int j = 0; j < 3; ++j) {
      M[0][j] = M[1][j]; G[0][j] = G[1][j];
      M[1][j] = M[2][j]; G[1][j] = G[2][j];
    }
#pragma unroll
    for (int k = 0; k + 1 < POOL_ROW_PF; ++k) {
      qm[k] = qm[k + 1];
      qg[k] = qg[k + 1];
    }
    qm[POOL_ROW_PF - 1] = nm;
    qg[POOL_ROW_PF - 1] = ng;
  }
}

// Stride-2 3x3 backward: a thread owns the 2x2 pixel block (h0, w0) = (2i - pad,
// 2j - pad) + {0,1}^2.  On the padded grid an even row is the bottom row of
// window i-1 and the top row of window i, an odd row the middle row of window
// i (same for columns), so the block is covered by exactly the windows
// (i-1, j-1), (i-1, j), (i, j-1), (i, j): one 8-byte shared load each and 9
// argmax tests for 4 pixels, visited in window raster order (bit-exact).
template <int CW>
__global__ void maxpool3s2_bwd_plane(const float* __restrict__ mask, const float* __restrict__ dy,
                                     float* __restrict__ dx, int planes, int G, int H, int W,
                                     int P, int Q, int pad, const float* __restrict__ relu_x) {
  extern __shared__ float2 pairs_all[];
  const int64_t pl0 = (int64_t)blockIdx.x * G;
  const int g_here = (int)(planes - pl0 < G ? planes - pl0 : G);
  const int PQ = P * Q;
  stage_pairs(pairs_all, mask + pl0 * PQ, dy + pl0 * PQ, g_here * PQ);
  __syncthreads();
  constexpr int RPW = 32 / CW;
  const int BI = (H + pad + 1) / 2, BJ = (W + pad + 1) / 2;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  const int roff = lane / CW, col = lane % CW;
  for (int rr = warp * RPW + roff; rr < g_here * BI; rr += nw * RPW) {
    const int g = rr / BI, i = rr - g * BI;
    const float2* pr = pairs_all + g * PQ;
    const int64_t pbase = (pl0 + g) * (int64_t)H * W;
    float* dp = dx + pbase;
    const int h0 = 2 * i - pad;
    const bool r0 = h0 >= 0, r1 = h0 + 1 < H;  // block rows inside the plane
    const bool pa = i - 1 >= 0 && i - 1 < P, pb = i < P;
    const int rowa = (pa ? i - 1 : 0) * Q, rowb = (pb ? i : 0) * Q;
    for (int j = col; j < BJ; j += CW) {
      const int w0 = 2 * j - pad;
      const bool qa = j - 1 >= 0 && j - 1 < Q, qb = j < Q;
      const float2 wAA = pr[rowa + (qa ? j - 1 : 0)];
      const float2 wAB = pr[rowa + (qb ? j : 0)];
      const float2 wBA = pr[rowb + (qa ? j - 1 : 0)];
      const float2 wBB = pr[rowb + (qb ? j : 0)];
      const float e00 = (float)(h0 * W + w0);
      const float e01 = e00 + 1.f, e10 = e00 + (float)W, e11 = e10 + 1.f;
      float a00 = 0.f, a01 = 0.f, a10 = 0.f, a11 = 0.f;
      // window (i-1, j-1): pixel (0,0)
      a00 = __fadd_rn(a00, (pa && qa && wAA.x == e00) ? wAA.y : 0.f);
      // window (i-1, j): pixels (0,0), (0,1)
      a00 = __fadd_rn(a00, (pa && qb && wAB.x == e00) ? wAB.y : 0.f);
      a01 = __fadd_rn(a01, (pa && qb && wAB.x == e01) ? wAB.y : 0.f);
      // window (i, j-1): pixels (0,0), (1,0)
      a00 = __fadd_rn(a00, (pb && qa && wBA.x == e00) ? wBA.y : 0.f);
      a10 = __fadd_rn(a10, (pb && qa && wBA.x == e10) ? wBA.y : 0.f);
      // window (i, j): all four
      const bool bb = pb && qb;
      a00 = __fadd_rn(a00, (bb && wBB.x == e00) ? wBB.y : 0.f);
      a01 = __fadd_rn(a01, (bb && wBB.x == e01) ? wBB.y : 0.f);
      a10 = __fadd_rn(a10, (bb && wBB.x == e10) ? wBB.y : 0.f);
      a11 = __fadd_rn(a11, (bb && wBB.x == e11) ? wBB.y : 0.f);
      const bool c0 = w0 >= 0, c1 = w0 + 1 < W;
      const int64_t o00 = (int64_t)h0 * W + w0, o10 = o00 + W;
      if (r0) {
        if (c0) dp[o00] = relu_fold(relu_x, pbase + o00, a00);
        if (c1) dp[o00 + 1] = relu_fold(relu_x, pbase + o00 + 1, a01);
      }
      if (r1) {
        if (c0) dp[o10] = relu_fold(relu_x, pbase + o10, a10);
        if (c1) dp[o10 + 1] = relu_fold(relu_x, pbase + o10 + 1, a11);
      }
    }
  }
}

// LRN, one thread per (n, V consecutive pixels) walking the channels with a
// 5-wide register window (size == 5, the GoogLeNet / AlexNet setting): every
// input element is loaded exactly once (V = 4: 16-byte loads and stores).
// Out-of-range window slots hold +0.0, which leaves the in-order sums unchanged.
#ifndef LRN_VEC
#define LRN_VEC 4
#endif
template <int V>
struct Vec;
template <>
struct Vec<1> {
  __device__ static void ld(const float* p, float (&v)[1]) { v[0] = __ldg(p); }
  __device__ static void st(float* p, const float (&v)[1]) { *p = v[0]; }
};
template <>
struct Vec<2> {
  __device__ static void ld(const float* p, float (&v)[2]) {
    const float2 f = __ldg(reinterpret_cast<const float2*>(p));
    v[0] = f.x; v[1] = f.y;
  }
  __device__ static void st(float* p, const float (&v)[2]) {
    *reinterpret_cast<float2*>(p) = make_float2(v[0], v[1]);
  }
};
template <>
struct Vec<4> {
  __device__ static void ld(const float* p, float (&v)[4]) {
    const float4 f = __ldg(reinterpret_cast<const float4*>(p));
    v[0] = f.x; v[1] = f.y; v[2] = f.z; v[3] = f.w;
  }
  __device__ static void st(float* p, const float (&v)[4]) {
    *reinterpret_cast<float4*>(p) = make_float4(v[0], v[1], v[2], v[3]);
  }
};

// backward: x, y, scale and dy each loaded once (y as given: the operator's
// contract, ops-level, takes the forward output as an input); the power is
// shared between the entering element's ratio and its later centre term.
template <int V>
__global__ void lrn5_bwd_kernel(const float* __restrict__ x, const float* __restrict__ y,
                                const float* __restrict__ scale, const float* __restrict__ dy,
                                float* __restrict__ dx, int N, int C, int HW, float coef,
                                float beta, int CH, const float* __restrict__ relu_x) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int HWV = HW / V;
  if (t >= (int64_t)N * HWV) return;
  const int n = (int)(t / HWV), hw = (int)(t - (int64_t)n * HWV) * V;
  const int64_t base = (int64_t)n * C * HW + hw;
  const int c0 = blockIdx.y * CH, c1 = min(C, c0 + CH);
  // r[0..4] = ratio[c-2 .. c+2] = dy*y/scale;  for c..c+2 also x, dy, scale^-beta
  float r[5][V], xs[3][V], ds[3][V], pw[3][V];
  auto enter = [&](int j, float (&xv)[V], float (&dv)[V], float (&pv)[V], float (&rv)[V]) {
    float sv[V], yv[V];
    Vec<V>::ld(x + base + (int64_t)j * HW, xv);
    Vec<V>::ld(y + base + (int64_t)j * HW, yv);
    Vec<V>::ld(dy + base + (int64_t)j * HW, dv);
    Vec<V>::ld(scale + base + (int64_t)j * HW, sv);
#pragma unroll
    for (int v = 0; v < V; ++v) {
      pv[v] = lrn_pow(sv[v], -beta);
      rv[v] = lrn_div(__fmul_rn(dv[v], yv[v]), sv[v]);
    }
  };
  // halo channels c0-2, c0-1: only their ratios
#pragma unroll
  for (int j = 0; j < 2; ++j) {
    const int c = c0 - 2 + j;
    if (c >= 0) {
      float sv[V], yv[V], dv[V];
      Vec<V>::ld(y + base + (int64_t)c * HW, yv);
      Vec<V>::ld(dy + base + (int64_t)c * HW, dv);
      Vec<V>::ld(scale + base + (int64_t)c * HW, sv);
#pragma unroll
      for (int v = 0; v < V; ++v) r[j][v] = lrn_div(__fmul_rn(dv[v], yv[v]), sv[v]);
    } else {
#pragma unroll
      for (int v = 0; v < V; ++v) r[j][v] = 0.f;
    }
  }
#pragma unroll
  for (int j = 0; j < 3; ++j) {
    if (c0 + j < C) {
      enter(c0 + j, xs[j], ds[j], pw[j], r[2 + j]);
    } else {
#pragma unroll
      for (int v = 0; v < V; ++v) xs[j][v] = ds[j][v] = pw[j][v] = r[2 + j][v] = 0.f;
    }
  }
  for (int c = c0; c < c1; ++c) {
    float out[V];
#pragma unroll
    for (int v = 0; v < V; ++v) {
      float acc = 0.f;
      acc = __fadd_rn(acc, r[0][v]);
      acc = __fadd_rn(acc, r[1][v]);
      acc = __fadd_rn(acc, r[2][v]);
      acc = __fadd_rn(acc, r[3][v]);
      acc = __fadd_rn(acc, r[4][v]);
      const float a = __fmul_rn(ds[0][v], pw[0][v]);
      const float b = __fmul_rn(__fmul_rn(coef, xs[0][v]), acc);
      out[v] = __fsub_rn(a, b);
    }
    if (relu_x) {
      float rx[V];
      Vec<V>::ld(relu_x + base + (int64_t)c * HW, rx);
#pragma unroll
      for (int v = 0; v < V; ++v) out[v] = rx[v] > 0.f ? out[v] : 0.f;
    }
    Vec<V>::st(dx + base + (int64_t)c * HW, out);
    float xn[V], dn[V], pn[V], rn[V];
    if (c + 3 < C) {
      enter(c + 3, xn, dn, pn, rn);
    } else {
#pragma unroll
      for (int v = 0; v < V; ++v) xn[v] = dn[v] = pn[v] = rn[v] = 0.f;
    }
#pragma unroll
    for (int v = 0; v < V; ++v) {
      r[0][v] = r[1][v];
      r[1][v] = r[2][v];
      r[2][v] = r[3][v];
      r[3][v] = r[4][v];
      r[4][v] = rn[v];
      xs[0][v] = xs[1][v]; xs[1][v] = xs[2][v]; xs[2][v] = xn[v];
      ds[0][v] = ds[1][v]; ds[1][v] = ds[2][v]; ds[2][v] = dn[v];
      pw[0][v] = pw[1][v]; pw[1][v] = pw[2][v]; pw[2][v] = pn[v];
    }
  }
}

#ifndef LRN_RC_VEC
#define LRN_RC_VEC 2
#endif

// The graph-plan LRN pair.  Forward: y (and scale unless the plan elides it),
// with x loads issued two channels ahead of their use.  Backward: scale and y
// are RECOMPUTED from x with the forward's exact operation sequence (same
// window order, same lrn_pow), so the result is bit-identical to the explicit
// backward fed with the forward's outputs, while reading only x and dy (plus
// the folded ReLU mask): 3-4 tensors of traffic per element instead of 6.
template <int V>
__device__ __forceinline__ void lrn_ld(const float* p, bool ok, float (&v)[V]) {
  if (ok) {
    Vec<V>::ld(p, v);
  } else {
#pragma unroll
    for (int i = 0; i < V; ++i) v[i] = 0.f;
  }
}

template <int V>
__device__ __forceinline__ float lrn_scale5(const float (&xq)[5][V], int v, float a_n, float kk) {
  float acc = 0.f;
#pragma unroll
  for (int j = 0; j < 5; ++j) acc = __fadd_rn(acc, __fmul_rn(xq[j][v], xq[j][v]));
  return __fadd_rn(kk, __fmul_rn(a_n, acc));
}

template <int V>
__global__ void __launch_bounds__(256) lrn5_fwd_pf_kernel(const float* __restrict__ x,
                                                          float* __restrict__ y,
                                                          float* __restrict__ scale, int N, int C,
                                                          int HW, float a_n, float beta, float kk,
                                                          int CH) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int HWV = HW / V;
  if (t >= (int64_t)N * HWV) return;
  const int n = (int)(t / HWV), hw = (int)(t - (int64_t)n * HWV) * V;
  const float* xb = x + (int64_t)n * C * HW + hw;
  const int64_t ob = (int64_t)n * C * HW + hw;
  const int c0 = blockIdx.y * CH, c1 = min(C, c0 + CH);
  float xq[5][V], xn[2][V];  // x[c-2 .. c+2], then x[c+3], x[c+4]
#pragma unroll
  for (int j = 0; j < 5; ++j) lrn_ld<V>(xb + (int64_t)(c0 - 2 + j) * HW, c0 - 2 + j >= 0 && c0 - 2 + j < C, xq[j]);
#pragma unroll
  for (int j = 0; j < 2; ++j) lrn_ld<V>(xb + (int64_t)(c0 + 3 + j) * HW, c0 + 3 + j < C, xn[j]);
  for (int c = c0; c < c1; ++c) {
    float xl[V];
    lrn_ld<V>(xb + (int64_t)(c + 5) * HW, c + 5 < C, xl);
    float sc[V], yv[V];
#pragma unroll
    for (int v = 0; v < V; ++v) {
      sc[v] = lrn_scale5<V>(xq, v, a_n, kk);
      yv[v] = __fmul_rn(xq[2][v], lrn_pow(sc[v], -beta));
    }
    if (scale) Vec<V>::st(scale + ob + (int64_t)c * HW, sc);
    Vec<V>::st(y + ob + (int64_t)c * HW, yv);
#pragma unroll
    for (int v = 0; v < V; ++v) {
      xq[0][v] = xq[1][v]; xq[1][v] = xq[2][v]; xq[2][v] = xq[3][v]; xq[3][v] = xq[4][v];
      xq[4][v] = xn[0][v]; xn[0][v] = xn[1][v]; xn[1][v] = xl[v];
    }
  }
}

template <int V>
__global__ void __launch_bounds__(256) lrn5_bwd_rc_kernel(const float* __restrict__ x,
                                                          const float* __restrict__ dy,
                                                          float* __restrict__ dx, int N, int C,
                                                          int HW, float a_n, float kk, float coef,
                                                          float beta, int CH,
                                                          const float* __restrict__ relu_x) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int HWV = HW / V;
  if (t >= (int64_t)N * HWV) return;
  const int n = (int)(t / HWV), hw = (int)(t - (int64_t)n * HWV) * V;
  const int64_t base = (int64_t)n * C * HW + hw;
  const float* xb = x + base;
  const float* db = dy + base;
  const int c0 = blockIdx.y * CH, c1 = min(C, c0 + CH);
  // iteration c enters channel e = c + 2 (its scale, scale^-beta and ratio
  // dy*y/scale) and, for c >= c0, emits dx[c].  State at the top of iteration c:
  //   xq = x[c .. c+4], dq = dy[c .. c+2], pq = pw[c-1 .. c+1], r = ratio[c-3 .. c+1]
  //   prefetched: xn = x[c+5], x[c+6]; dn = dy[c+3], dy[c+4]
  float xq[5][V], dq[3][V], pq[3][V], r[5][V], xn[2][V], dn[2][V];
  const int cs = c0 - 4;
#pragma unroll
  for (int j = 0; j < 5; ++j) lrn_ld<V>(xb + (int64_t)(cs + j) * HW, cs + j >= 0 && cs + j < C, xq[j]);
#pragma unroll
  for (int j = 0; j < 3; ++j) lrn_ld<V>(db + (int64_t)(cs + j) * HW, cs + j >= 0 && cs + j < C, dq[j]);
#pragma unroll
  for (int j = 0; j < 2; ++j) {
    lrn_ld<V>(xb + (int64_t)(cs + 5 + j) * HW, cs + 5 + j >= 0 && cs + 5 + j < C, xn[j]);
    lrn_ld<V>(db + (int64_t)(cs + 3 + j) * HW, cs + 3 + j >= 0 && cs + 3 + j < C, dn[j]);
  }
#pragma unroll
  for (int v = 0; v < V; ++v) {
#pragma unroll
    for (int j = 0; j < 5; ++j) r[j][v] = 0.f;
#pragma unroll
    for (int j = 0; j < 3; ++j) pq[j][v] = 0.f;
  }
  for (int c = cs; c < c1; ++c) {
    float xl[V], dl[V], rx[V];
    lrn_ld<V>(xb + (int64_t)(c + 7) * HW, c + 7 >= 0 && c + 7 < C, xl);
    lrn_ld<V>(db + (int64_t)(c + 5) * HW, c + 5 >= 0 && c + 5 < C, dl);
    const bool emit = c >= c0;
    // relu_x == x: the folded ReLU's mask is x's own sign (x is that ReLU's
    // output: relu(a) > 0 <=> a > 0), already in registers as xq[0]
    const bool own = relu_x == x;
    if (relu_x && !own && emit) Vec<V>::ld(relu_x + base + (int64_t)c * HW, rx);
    const bool live = c + 2 >= 0 && c + 2 < C;
#pragma unroll
    for (int v = 0; v < V; ++v) {
      float pe = 0.f, re = 0.f;
      if (live) {
        const float s = lrn_scale5<V>(xq, v, a_n, kk);
        pe = lrn_pow(s, -beta);
        const float ye = __fmul_rn(xq[2][v], pe);
        re = lrn_div(__fmul_rn(dq[2][v], ye), s);
      }
      r[0][v] = r[1][v]; r[1][v] = r[2][v]; r[2][v] = r[3][v]; r[3][v] = r[4][v]; r[4][v] = re;
      pq[0][v] = pq[1][v]; pq[1][v] = pq[2][v]; pq[2][v] = pe;
    }
    if (emit) {
      float out[V];
#pragma unroll
      for (int v = 0; v < V; ++v) {
        float acc = 0.f;
        acc = __fadd_rn(acc, r[0][v]);
        acc = __fadd_rn(acc, r[1][v]);
        acc = __fadd_rn(acc, r[2][v]);
        acc = __fadd_rn(acc, r[3][v]);
        acc = __fadd_rn(acc, r[4][v]);
        const float a = __fmul_rn(dq[0][v], pq[0][v]);
        const float b = __fmul_rn(__fmul_rn(coef, xq[0][v]), acc);
        out[v] = __fsub_rn(a, b);
        if (relu_x) out[v] = (own ? xq[0][v] : rx[v]) > 0.f ? out[v] : 0.f;
      }
      Vec<V>::st(dx + base + (int64_t)c * HW, out);
    }
#pragma unroll
    for (int v = 0; v < V; ++v) {
      xq[0][v] = xq[1][v]; xq[1][v] = xq[2][v]; xq[2][v] = xq[3][v]; xq[3][v] = xq[4][v];
      xq[4][v] = xn[0][v]; xn[0][v] = xn[1][v]; xn[1][v] = xl[v];
      dq[0][v] = dq[1][v]; dq[1][v] = dq[2][v]; dq[2][v] = dn[0][v];
      dn[0][v] = dn[1][v]; dn[1][v] = dl[v];
    }
  }
}

// channel chunk for the LRN walkers: enough (pixel group, chunk) threads to
// fill the GPU several times over; each chunk re-reads a 2-channel halo
static int lrn_chunk(int64_t pixel_threads, int C) {
  const int64_t want = (int64_t)sm_count_current() * 2048 * 2;
  int chunks = (int)std::min<int64_t>(std::max<int64_t>(1, want / std::max<int64_t>(1, pixel_threads)),
                                      (C + 15) / 16);
  return (C + chunks - 1) / chunks;
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

// vector width for the graph-plan LRN kernels: LRN_RC_VEC when the plane size
// and every pointer allow it, else scalar
static int lrn_vec(int HW, std::initializer_list<const void*> ptrs) {
  int v = LRN_RC_VEC;
  while (v > 1) {
    bool ok = HW % v == 0;
    for (const void* p : ptrs) ok = ok && ((uintptr_t)p % (4u * v)) == 0;
    if (ok) break;
    v /= 2;
  }
  return v;
}

template <int V>
static void lrn5_fwd_launch(const float* x, float* y, float* scale, int N, int C, int HW,
                            float a_n, float beta, float k, cudaStream_t st) {
  const int64_t px = (int64_t)N * HW / V;
  const int ch = lrn_chunk(px, C);
  lrn5_fwd_pf_kernel<V><<<dim3((unsigned)((px + 255) / 256), (C + ch - 1) / ch), 256, 0, st>>>(
      x, y, scale, N, C, HW, a_n, beta, k, ch);
}

template <int V>
static void lrn5_bwd_rc_launch(const float* x, const float* dy, float* dx, const float* relu_x,
                               int N, int C, int HW, float a_n, float k, float coef, float beta,
                               cudaStream_t st) {
  const int64_t px = (int64_t)N * HW / V;
  const int ch = lrn_chunk(px, C);
  lrn5_bwd_rc_kernel<V><<<dim3((unsigned)((px + 255) / 256), (C + ch - 1) / ch), 256, 0, st>>>(
      x, dy, dx, N, C, HW, a_n, k, coef, beta, ch, relu_x);
}

// column walkers on/off (A/B): bit 0 forward stride 1, bit 1 forward stride 2,
// bit 2 backward stride 1, bit 3 warp-row kernels (stride 1, pad 1, W <= 32);
// PURINE_B200_POOL_WALKERS, default all on
static int pool_walkers() {
  // bit 0/1: stride-1/2 column walkers, 2: stride-1 backward walker, 3: warp-row
  // kernels, 4: shared-memory staged forward, 5: staged mask-reading backward
  // (pool_staged.cu)
  const char* e = std::getenv("PURINE_B200_POOL_WALKERS");
  return e ? std::atoi(e) : 63;
}

extern "C" {

int bf_maxpool_fwd(const float* x, float* y, float* mask, int N, int C, int H, int W, int P,
                   int Q, int kernel, int stride, int pad, bf_stream_t s) {
  int64_t total = (int64_t)N * C * P * Q;
  if (total <= 0) return 0;
  // staged through shared memory by bulk copies (pool_staged.cu) where it fits
  if ((pool_walkers() & 16) && (reinterpret_cast<uintptr_t>(x) & 15) == 0 &&
      bf_maxpool_staged_ok(N, C, H, W, P, Q, kernel, stride, pad, 0))
    return bf_maxpool_fwd_staged(x, y, mask, N, C, H, W, P, Q, kernel, stride, pad, s);
  if (kernel == 3 && stride == 1 && pad == 1 && W <= 32 && P == H && Q == W &&
      (pool_walkers() & 8)) {
    const int64_t planes = (int64_t)N * C, warps = (planes + 32 / W - 1) / (32 / W);
    maxpool3s1_fwd_rows<<<(unsigned)((warps + 7) / 8), 256, 0, as_stream(s)>>>(x, y, mask, planes,
                                                                               H, W);
    return check_launch("maxpool_forward");
  }
  if (kernel == 3 && (stride == 1 || stride == 2) && (pool_walkers() >> (stride - 1)) & 1) {
    const int64_t threads = (int64_t)N * C * Q;
    const unsigned blocks = (unsigned)((threads + 255) / 256);
    if (stride == 1)
      maxpool3_fwd_cols<1><<<blocks, 256, 0, as_stream(s)>>>(x, y, mask, threads, H, W, P, Q, pad);
    else
      maxpool3_fwd_cols<2><<<blocks, 256, 0, as_stream(s)>>>(x, y, mask, threads, H, W, P, Q, pad);
    return check_launch("maxpool_forward");
  }
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
  return bf_maxpool_bwd_relu(mask, dy, dx, nullptr, N, C, H, W, P, Q, kernel, stride, pad, s);
}

int bf_maxpool_bwd_relu(const float* mask, const float* dy, float* dx, const float* relu_x, int N,
                        int C, int H, int W, int P, int Q, int kernel, int stride, int pad,
                        bf_stream_t s) {
  int64_t total = (int64_t)N * C * H * W;
  if (total <= 0) return 0;
  // mask + dy staged through shared memory (pool_staged.cu) where it fits
  if (!relu_x && (pool_walkers() & 32) &&
      ((reinterpret_cast<uintptr_t>(mask) | reinterpret_cast<uintptr_t>(dy)) & 15) == 0 &&
      bf_maxpool_staged_ok(N, C, H, W, P, Q, kernel, stride, pad, 2))
    return bf_maxpool_bwd_staged(mask, dy, dx, N, C, H, W, P, Q, kernel, stride, pad, s);
  if (kernel == 3 && stride == 1 && pad == 1 && W <= 32 && P == H && Q == W &&
      (pool_walkers() & 8)) {
    const int64_t planes = (int64_t)N * C, warps = (planes + 32 / W - 1) / (32 / W);
    maxpool3s1_bwd_rows<<<(unsigned)((warps + 7) / 8), 256, 0, as_stream(s)>>>(
        mask, dy, dx, planes, H, W, relu_x);
    return check_launch("maxpool_backward");
  }
  if (kernel == 3 && stride == 1 && (pool_walkers() & 4)) {
    const int64_t threads = (int64_t)N * C * W;
    maxpool3s1_bwd_cols<<<(unsigned)((threads + 255) / 256), 256, 0, as_stream(s)>>>(
        mask, dy, dx, threads, H, W, P, Q, pad, relu_x);
    return check_launch("maxpool_backward");
  }
  const int smem = 2 * P * Q * 4;
  if (smem <= kPlaneSmemMax) {
    static bool attr = false;
    if (!attr) {
      BF_CUDA(cudaFuncSetAttribute(maxpool_bwd_plane, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   kPlaneSmemMax),
              "maxpool smem attribute");
      const void* fns[] = {(const void*)maxpool3s2_bwd_plane<8>,
                           (const void*)maxpool3s2_bwd_plane<16>,
                           (const void*)maxpool3s2_bwd_plane<32>,
                           (const void*)maxpool3_bwd_plane<1, 8>,
                           (const void*)maxpool3_bwd_plane<1, 16>,
                           (const void*)maxpool3_bwd_plane<1, 32>};
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
  maxpool3_bwd_plane<SS, CC><<<blocks, 256, sm, as_stream(s)>>>(mask, dy, dx, planes, G, H, W, P, Q, pad, relu_x)
      if (stride == 1) {
        if (cw == 8) BF_MP3B(1, 8); else if (cw == 16) BF_MP3B(1, 16); else BF_MP3B(1, 32);
      } else {
        const int bj = (W + pad + 1) / 2;
        const int cw2 = bj <= 8 ? 8 : (bj <= 16 ? 16 : 32);
#define BF_MP3B2(CC)                                                                            \
  maxpool3s2_bwd_plane<CC><<<blocks, 256, sm, as_stream(s)>>>(mask, dy, dx, planes, G, H, W, P, \
                                                              Q, pad, relu_x)
        if (cw2 == 8) BF_MP3B2(8); else if (cw2 == 16) BF_MP3B2(16); else BF_MP3B2(32);
#undef BF_MP3B2
      }
#undef BF_MP3B
      return check_launch("maxpool_backward");
    }
    maxpool_bwd_plane<<<N * C, 256, smem, as_stream(s)>>>(mask, dy, dx, H, W, P, Q, kernel,
                                                          stride, pad, relu_x);
    return check_launch("maxpool_backward");
  }
  maxpool_bwd_kernel<<<elementwise_grid(total, kThreads), kThreads, 0, as_stream(s)>>>(
      mask, dy, dx, total, H, W, P, Q, kernel, stride, pad, relu_x);
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
  if (P == 1 && Q == 1 && pad == 0 && kernel == H && kernel == W && total < (1LL << 31)) {
    avgpool_global_bwd_kernel<<<elementwise_grid(total, kThreads), kThreads, 0, as_stream(s)>>>(
        dy, dx, (uint32_t)total, (uint32_t)(H * W), (float)(H * W));
    return check_launch("avgpool_backward");
  }
  avgpool_bwd_kernel<<<elementwise_grid(total, kThreads), kThreads, 0, as_stream(s)>>>(
      dy, dx, total, H, W, P, Q, kernel, stride, pad);
  return check_launch("avgpool_backward");
}

int bf_lrn_fwd(const float* x, float* y, float* scale, int N, int C, int H, int W, int size,
               float alpha, float beta, float k, bf_stream_t s) {
  BF_REQUIRE(size >= 1, "lrn_forward: size must be >= 1");
  BF_REQUIRE(scale || size == 5, "lrn_forward: scale may be omitted only for size 5");
  int64_t total = (int64_t)N * C * H * W;
  if (total <= 0) return 0;
  int pre = (size - 1) / 2, post = size - 1 - pre;
  float a_n = alpha / (float)size;
  if (size == 5) {
    const int HW = H * W;
    switch (lrn_vec(HW, {x, y, scale})) {
      case 4: lrn5_fwd_launch<4>(x, y, scale, N, C, HW, a_n, beta, k, as_stream(s)); break;
      case 2: lrn5_fwd_launch<2>(x, y, scale, N, C, HW, a_n, beta, k, as_stream(s)); break;
      default: lrn5_fwd_launch<1>(x, y, scale, N, C, HW, a_n, beta, k, as_stream(s)); break;
    }
    return check_launch("lrn_forward");
  }
  lrn_fwd_kernel<<<elementwise_grid(total, kThreads), kThreads, 0, as_stream(s)>>>(
      x, y, scale, total, C, H * W, pre, post, a_n, beta, k);
  return check_launch("lrn_forward");
}

int bf_lrn_bwd_recompute(const float* x, const float* dy, float* dx, const float* relu_x, int N,
                         int C, int H, int W, int size, float alpha, float beta, float k,
                         bf_stream_t s) {
  BF_REQUIRE(size == 5, "lrn_backward (recompute): size must be 5");
  if ((int64_t)N * C * H * W <= 0) return 0;
  const float a_n = alpha / (float)size;
  float coef = 2.0f * alpha;
  coef = coef * beta;
  coef = coef / (float)size;
  const int HW = H * W;
  switch (lrn_vec(HW, {x, dy, dx, relu_x})) {
    case 4: lrn5_bwd_rc_launch<4>(x, dy, dx, relu_x, N, C, HW, a_n, k, coef, beta, as_stream(s)); break;
    case 2: lrn5_bwd_rc_launch<2>(x, dy, dx, relu_x, N, C, HW, a_n, k, coef, beta, as_stream(s)); break;
    default: lrn5_bwd_rc_launch<1>(x, dy, dx, relu_x, N, C, HW, a_n, k, coef, beta, as_stream(s)); break;
  }
  return check_launch("lrn_backward");
}

int bf_lrn_bwd(const float* x, const float* y, const float* scale, const float* dy, float* dx,
               int N, int C, int H, int W, int size, float alpha, float beta, float k,
               bf_stream_t s) {
  return bf_lrn_bwd_relu(x, y, scale, dy, dx, nullptr, N, C, H, W, size, alpha, beta, k, s);
}

int bf_lrn_bwd_relu(const float* x, const float* y, const float* scale, const float* dy,
                    float* dx, const float* relu_x, int N, int C, int H, int W, int size,
                    float alpha, float beta, float k, bf_stream_t s) {
  BF_REQUIRE(size >= 1, "lrn_backward: size must be >= 1");
  int64_t total = (int64_t)N * C * H * W;
  if (total <= 0) return 0;
  int pre = (size - 1) / 2, post = size - 1 - pre;
  float coef = 2.0f * alpha;
  coef = coef * beta;
  coef = coef / (float)size;
  if (size == 5) {
    int64_t px = (int64_t)N * H * W;
    if (LRN_VEC == 4 && (H * W) % 4 == 0 &&
        (((uintptr_t)x | (uintptr_t)y | (uintptr_t)scale | (uintptr_t)dy | (uintptr_t)dx |
          (uintptr_t)relu_x) & 15) == 0)
    {
      const int ch = lrn_chunk(px / 4, C);
      lrn5_bwd_kernel<4><<<dim3((unsigned)((px / 4 + 255) / 256), (C + ch - 1) / ch), 256, 0,
                           as_stream(s)>>>(x, y, scale, dy, dx, N, C, H * W, coef, beta, ch,
                                           relu_x);
    } else {
      const int ch = lrn_chunk(px, C);
      lrn5_bwd_kernel<1><<<dim3((unsigned)((px + 255) / 256), (C + ch - 1) / ch), 256, 0,
                           as_stream(s)>>>(x, y, scale, dy, dx, N, C, H * W, coef, beta, ch,
                                           relu_x);
    }
    return check_launch("lrn_backward");
  }
  lrn_bwd_kernel<<<elementwise_grid(total, kThreads), kThreads, 0, as_stream(s)>>>(
      x, y, scale, dy, dx, total, C, H * W, pre, post, coef, beta, relu_x);
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
