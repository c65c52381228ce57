// Implicit-GEMM operand loaders and epilogues shared by the GEMM engines.
//
// Every dense contraction on the path is expressed as
//     D[m][n] = sum_k A(m, k) * B(n, k)
// with A and B read straight out of the reference's NCHW / KCRS / row-major
// tensors by a loader (no materialised im2col):
//
//   pass            M            N        K            A(m,k)            B(n,k)
//   conv fwd        N*P*Q pix    Kout     C*R*S        x gathered        w[kout][crs]
//   conv dgrad      N*H*W pix    C        Kout*R*S     dy gathered       w[kout][c][r][s]
//   conv wgrad      C*R*S        Kout     N*P*Q        x gathered        dy[n][kout][pq]
//   fc fwd          m (units)    n        d            w[d][m]           x[n][d]
//   fc dgrad        d            n        m            w[d][m]           dy[n][m]
//   fc wgrad        m            d        n            dy[n][m]          x[n][d]
//
// The M index is always the one contiguous in the OUTPUT, so epilogue stores
// are coalesced along m.  Which index is contiguous in the INPUT decides the
// loader's thread mapping (kMContig).
#pragma once

#include <algorithm>

#include "common.cuh"

namespace bf {

struct ConvShape {
  int N, C, H, W, K, R, S, P, Q, stride, pad;
};

// ---- A / B loaders --------------------------------------------------------

// conv fwd A: row = output pixel (n,p,q), k = (c,r,s)
struct LdFwdX {
  static constexpr bool kMContig = true;
  const float* x;
  ConvShape g;
  __device__ __forceinline__ float operator()(int m, int k) const {
    int PQ = g.P * g.Q, RS = g.R * g.S;
    int n = m / PQ, pq = m - n * PQ;
    int p = pq / g.Q, q = pq - p * g.Q;
    int c = k / RS, rs = k - c * RS;
    int r = rs / g.S, s = rs - r * g.S;
    int ih = p * g.stride - g.pad + r, iw = q * g.stride - g.pad + s;
    if ((unsigned)ih >= (unsigned)g.H || (unsigned)iw >= (unsigned)g.W) return 0.f;
    return x[(((int64_t)n * g.C + c) * g.H + ih) * g.W + iw];
  }
};

// row-major [rows][ld] with k along the row (K-contiguous)
struct LdRowK {
  static constexpr bool kMContig = false;
  const float* p;
  int64_t ld;
  __device__ __forceinline__ float operator()(int m, int k) const { return p[m * ld + k]; }
};

// element (m, k) at p[k*ld + m] (M-contiguous)
struct LdColK {
  static constexpr bool kMContig = true;
  const float* p;
  int64_t ld;
  __device__ __forceinline__ float operator()(int m, int k) const { return p[k * ld + m]; }
};

// conv dgrad A: row = input pixel (n,h,w), k = (kout,r,s)
struct LdDgradDY {
  static constexpr bool kMContig = true;
  const float* dy;
  ConvShape g;
  __device__ __forceinline__ float operator()(int m, int k) const {
    int HW = g.H * g.W, RS = g.R * g.S;
    int n = m / HW, hw = m - n * HW;
    int h = hw / g.W, w = hw - h * g.W;
    int ko = k / RS, rs = k - ko * RS;
    int r = rs / g.S, s = rs - r * g.S;
    int th = h + g.pad - r, tw = w + g.pad - s;
    if (th < 0 || tw < 0) return 0.f;
    int oh = th / g.stride, ow = tw / g.stride;
    if (oh * g.stride != th || ow * g.stride != tw || oh >= g.P || ow >= g.Q) return 0.f;
    return dy[(((int64_t)n * g.K + ko) * g.P + oh) * g.Q + ow];
  }
};

// conv dgrad B: row = input channel c, k = (kout,r,s) -> w[kout][c][r][s]
struct LdDgradW {
  static constexpr bool kMContig = false;
  const float* w;
  ConvShape g;
  __device__ __forceinline__ float operator()(int c, int k) const {
    int RS = g.R * g.S;
    int ko = k / RS, rs = k - ko * RS;
    return w[((int64_t)ko * g.C + c) * RS + rs];
  }
};

// conv wgrad A: row = (c,r,s), k = output pixel (n,p,q)
struct LdWgradX {
  static constexpr bool kMContig = false;
  const float* x;
  ConvShape g;
  __device__ __forceinline__ float operator()(int crs, int k) const {
    int PQ = g.P * g.Q, RS = g.R * g.S;
    int c = crs / RS, rs = crs - c * RS;
    int r = rs / g.S, s = rs - r * g.S;
    int n = k / PQ, pq = k - n * PQ;
    int p = pq / g.Q, q = pq - p * g.Q;
    int ih = p * g.stride - g.pad + r, iw = q * g.stride - g.pad + s;
    if ((unsigned)ih >= (unsigned)g.H || (unsigned)iw >= (unsigned)g.W) return 0.f;
    return x[(((int64_t)n * g.C + c) * g.H + ih) * g.W + iw];
  }
};

// conv wgrad B: row = kout, k = output pixel (n,p,q)
struct LdWgradDY {
  static constexpr bool kMContig = false;
  const float* dy;
  ConvShape g;
  __device__ __forceinline__ float operator()(int ko, int k) const {
    int PQ = g.P * g.Q;
    int n = k / PQ, pq = k - n * PQ;
    return dy[((int64_t)n * g.K + ko) * PQ + pq];
  }
};

// ---- epilogues --------------------------------------------------------------

// Epilogues store D[m][n] with a per-row base and a per-column stride, so a
// thread that owns row m computes its base once (row(m)) and then writes
// out[base + n*stride] (+ bias) per column (store(r, n, v)).
struct RowPtr {
  float* p;
  float bias_row;  // EpiT's per-row bias (0 if none)
  int64_t relu_delta = 0;  // EpiNCHW: element offset of the fused ReLU output
};

// relu_forward's arithmetic, np.maximum(v, 0): NaN propagates, -0 -> +0
// (ops.py:359-364; elementwise.cu relu1)
__device__ __forceinline__ float relu_value(float v) { return !(v <= 0.f) ? v : 0.f; }

// out[(img*Cout + n)*PQ + pq] = v (+ bias[n]);  m = img*PQ + pq.
// With relu_out set the epilogue also writes relu(v) there: the graph's
// following relu_forward is fused away (dispatcher fusion plan).
struct EpiNCHW {
  float* out;
  const float* bias;
  int PQ, Cout;
  float* relu_out = nullptr;
  // relu_out layout: image stride (elements) and first channel, so the ReLU
  // can land directly in a channel slice of a concatenated tensor
  int64_t relu_img = 0;  // 0: same layout as out
  int relu_c0 = 0;
  // relu_backward folded in (dgrad): out = (relu_x > 0 ? v : 0), relu_x laid out as out
  const float* relu_x = nullptr;
  // the pre-activation has no reader (dispatcher: every consumer is fused or
  // reads the ReLU output instead): only the ReLU output is stored.  `out`
  // is then only the base of the row arithmetic (never dereferenced)
  bool no_out = false;
  __device__ __forceinline__ void operator()(int m, int n, float v) const {
    int img = m / PQ, pq = m - img * PQ;
    if (bias) v = __fadd_rn(v, bias[n]);
    const int64_t o = ((int64_t)img * Cout + n) * PQ + pq;
    if (relu_x) v = relu_x[o] > 0.f ? v : 0.f;
    if (!no_out) out[o] = v;
    if (relu_out) relu_out[relu_index(img, pq) + (int64_t)n * PQ] = relu_value(v);
  }
  __device__ __forceinline__ int64_t relu_index(int img, int pq) const {
    return (relu_img ? (int64_t)img * relu_img : (int64_t)img * Cout * PQ) +
           (int64_t)relu_c0 * PQ + pq;
  }
  __device__ __forceinline__ RowPtr row(int m) const {
    int img = m / PQ, pq = m - img * PQ;
    float* base = out + (int64_t)img * Cout * PQ + pq;
    return {base, 0.f, relu_out ? (relu_out + relu_index(img, pq)) - base : 0};
  }
  __device__ __forceinline__ void store(const RowPtr& r, int n, float v) const {
    if (bias) v = __fadd_rn(v, __ldg(bias + n));
    float* p = r.p + (int64_t)n * PQ;
    if (relu_x) v = __ldg(relu_x + (p - out)) > 0.f ? v : 0.f;
    if (!no_out) *p = v;
    if (relu_out) p[r.relu_delta] = relu_value(v);
  }
  // 16 consecutive columns of one row (the tcgen05 epilogues).  Column j of
  // the row lives PQ elements after column j-1, so the address advances by a
  // constant; each optional feature is tested once per chunk (not per
  // element), full chunks skip the per-column bound, and the stores are
  // st.global.  (ncu, 1x1 data gradient: the per-element form cost ~28
  // instructions per output -- reloaded parameters, 64-bit multiplies, a
  // branch per column, generic stores -- 67% of the kernel's instructions.)
  __device__ __forceinline__ void store16(const RowPtr& r, int n0, const uint32_t (&v)[16],
                                          int nlim) const {
    const int64_t stride = PQ;
    float* p = r.p + (int64_t)n0 * stride;
    const float* rx = relu_x;
    const float* bs = bias;
    float* ro = relu_out;
    if (nlim >= 16 && !rx && !ro) {
      if (bs) {
        float b[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) b[j] = __ldg(bs + n0 + j);
#pragma unroll
        for (int j = 0; j < 16; ++j) __stcg(p + j * stride, __fadd_rn(__uint_as_float(v[j]), b[j]));
      } else {
#pragma unroll
        for (int j = 0; j < 16; ++j) __stcg(p + j * stride, __uint_as_float(v[j]));
      }
      return;
    }
    if (nlim >= 16 && !rx) {  // forward with the fused ReLU output
      const int64_t rd = r.relu_delta;
      if (no_out) {
        float b[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) b[j] = bs ? __ldg(bs + n0 + j) : 0.f;
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          float x = __uint_as_float(v[j]);
          if (bs) x = __fadd_rn(x, b[j]);
          __stcg(p + j * stride + rd, relu_value(x));
        }
        return;
      }
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        float x = __uint_as_float(v[j]);
        if (bs) x = __fadd_rn(x, __ldg(bs + n0 + j));
        __stcg(p + j * stride, x);
        __stcg(p + j * stride + rd, relu_value(x));
      }
      return;
    }
    if (nlim >= 16 && !bs && !ro) {  // data gradient with the ReLU backward folded in:
      // the folded ReLU's x values are all loaded before any store (overlap)
      const float* mx = rx + (p - out);
      float m[16];
#pragma unroll
      for (int j = 0; j < 16; ++j) m[j] = __ldg(mx + j * stride);
#pragma unroll
      for (int j = 0; j < 16; ++j) __stcg(p + j * stride, m[j] > 0.f ? __uint_as_float(v[j]) : 0.f);
      return;
    }
    // general form: partial chunk or an unusual feature mix
    float m[16];
    if (rx) {
      const float* mx = rx + (p - out);
#pragma unroll
      for (int j = 0; j < 16; ++j) m[j] = j < nlim ? __ldg(mx + j * stride) : 0.f;
    }
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      if (j >= nlim) continue;
      float x = __uint_as_float(v[j]);
      if (bs) x = __fadd_rn(x, __ldg(bs + n0 + j));
      if (rx) x = m[j] > 0.f ? x : 0.f;
      if (!no_out) __stcg(p + j * stride, x);
      if (ro) __stcg(p + j * stride + r.relu_delta, relu_value(x));
    }
  }
};

// Horizontally fused sibling convolutions (Inception's 1x1 / 3x3_reduce /
// 5x5_reduce reading the same x): one GEMM over the concatenated output
// channels; column n belongs to segment s with start[s] <= n < start[s + 1],
// whose output is out[s] (cout[s] channels, NCHW) with bias[s] and, if
// relu[s], relu(v) into channel relu_c0[s] + (n - start[s]) of a tensor with
// relu_img[s] elements per image.  RowPtr carries the row index m (relu_delta).
constexpr int kMaxSeg = 4;
struct EpiNCHWSeg {
  int PQ, nseg;
  int start[kMaxSeg + 1];
  float* out[kMaxSeg];
  const float* bias[kMaxSeg];
  int cout[kMaxSeg];
  float* relu[kMaxSeg];
  int64_t relu_img[kMaxSeg];
  int relu_c0[kMaxSeg];
  __device__ __forceinline__ int seg_of(int n) const {
    int s = 0;
#pragma unroll
    for (int i = 1; i < kMaxSeg; ++i) s += (i < nseg && n >= start[i]) ? 1 : 0;
    return s;
  }
  __device__ __forceinline__ void put(int img, int pq, int n, float v) const {
    const int s = seg_of(n), j = n - start[s];
    if (bias[s]) v = __fadd_rn(v, __ldg(bias[s] + j));
    if (out[s]) __stcg(out[s] + ((int64_t)img * cout[s] + j) * PQ + pq, v);
    if (relu[s]) __stcg(relu[s] + (int64_t)img * relu_img[s] + (int64_t)(relu_c0[s] + j) * PQ + pq,
                        relu_value(v));
  }
  __device__ __forceinline__ void operator()(int m, int n, float v) const {
    const int img = m / PQ;
    put(img, m - img * PQ, n, v);
  }
  __device__ __forceinline__ RowPtr row(int m) const { return {nullptr, 0.f, (int64_t)m}; }
  __device__ __forceinline__ void store16(const RowPtr& r, int n0, const uint32_t (&v)[16],
                                          int nlim) const {
    const int m = (int)r.relu_delta, img = m / PQ, pq = m - img * PQ;
    const int s = seg_of(n0);
    const int64_t stride = PQ;
    if (nlim >= 16 && n0 + 15 < start[s + 1]) {  // the chunk lies in one segment
      const int j0 = n0 - start[s];
      float* p = out[s] ? out[s] + ((int64_t)img * cout[s] + j0) * PQ + pq : nullptr;
      const float* bs = bias[s];
      float* rp = relu[s] ? relu[s] + (int64_t)img * relu_img[s] +
                                (int64_t)(relu_c0[s] + j0) * PQ + pq
                          : nullptr;
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        float x = __uint_as_float(v[j]);
        if (bs) x = __fadd_rn(x, __ldg(bs + j0 + j));
        if (p) __stcg(p + j * stride, x);
        if (rp) __stcg(rp + j * stride, relu_value(x));
      }
      return;
    }
#pragma unroll
    for (int j = 0; j < 16; ++j)
      if (j < nlim) put(img, pq, n0 + j, __uint_as_float(v[j]));
  }
};

// out[n*ldo + m] = v (+ bias[m])
struct EpiT {
  float* out;
  const float* bias;
  int64_t ldo;
  __device__ __forceinline__ void operator()(int m, int n, float v) const {
    if (bias) v = __fadd_rn(v, bias[m]);
    out[n * ldo + m] = v;
  }
  __device__ __forceinline__ RowPtr row(int m) const { return {out + m, bias ? bias[m] : 0.f}; }
  __device__ __forceinline__ void store(const RowPtr& r, int n, float v) const {
    if (bias) v = __fadd_rn(v, r.bias_row);
    r.p[n * ldo] = v;
  }
  __device__ __forceinline__ void store16(const RowPtr& r, int n0, const uint32_t (&v)[16],
                                          int nlim) const {
    float* p = r.p + (int64_t)n0 * ldo;
    if (bias) {  // (no bias: the value is stored as is, -0 included)
      const float b = r.bias_row;
#pragma unroll
      for (int j = 0; j < 16; ++j)
        if (j < nlim) __stcg(p + j * ldo, __fadd_rn(__uint_as_float(v[j]), b));
    } else if (nlim >= 16) {
#pragma unroll
      for (int j = 0; j < 16; ++j) __stcg(p + j * ldo, __uint_as_float(v[j]));
    } else {
#pragma unroll
      for (int j = 0; j < 16; ++j)
        if (j < nlim) __stcg(p + j * ldo, __uint_as_float(v[j]));
    }
  }
};

// split-K partial: ws[split][n][m]
struct EpiPartial {
  float* ws;
  int M, N;
  __device__ __forceinline__ void operator()(int split, int m, int n, float v) const {
    ws[((int64_t)split * N + n) * M + m] = v;
  }
  __device__ __forceinline__ RowPtr row(int split, int m) const {
    return {ws + (int64_t)split * N * M + m, 0.f};
  }
  __device__ __forceinline__ void store(const RowPtr& r, int n, float v) const {
    r.p[(int64_t)n * M] = v;
  }
  __device__ __forceinline__ void store16(const RowPtr& r, int n0, const uint32_t (&v)[16],
                                          int nlim) const {
    const int64_t stride = M;
    float* p = r.p + (int64_t)n0 * stride;
    if (nlim >= 16) {
#pragma unroll
      for (int j = 0; j < 16; ++j) __stcg(p + j * stride, __uint_as_float(v[j]));
      return;
    }
#pragma unroll
    for (int j = 0; j < 16; ++j)
      if (j < nlim) __stcg(p + j * stride, __uint_as_float(v[j]));
  }
};

// splits summed in order, then the final epilogue
template <class Epi>
__global__ void splitk_reduce_kernel(const float* __restrict__ ws, int splits, int M, int N,
                                     Epi epi) {
  int64_t total = (int64_t)M * N;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    float acc = ws[i];
    for (int s = 1; s < splits; ++s) acc = __fadd_rn(acc, ws[s * total + i]);
    int n = (int)(i / M), m = (int)(i - (int64_t)n * M);
    epi(m, n, acc);
  }
}

// many splits (chain-bounded weight gradients): thread (quad, g) sums the
// float4 of outputs [4*quad, 4*quad + 4) over splits g, g + G, g + 2G, ... in
// order (4 loads in flight per step), then the g = 0 threads add the G group
// sums in order -- a fixed summation tree, so the result is deterministic.
// G (a power of two <= 32) is sized so that even a small output (conv1's
// 9.4k weights over ~800 splits) keeps every SM streaming.
template <class Epi>
__global__ void __launch_bounds__(256) splitk_reduce_vec_kernel(const float* __restrict__ ws,
                                                                int splits, int M, int N, int G,
                                                                Epi epi) {
  __shared__ float4 part[256];
  const int64_t total = (int64_t)M * N, quads = total / 4;
  const int Q = 256 / G;
  const int t = threadIdx.x, quad_l = t % Q, g = t / Q;
  const float4* w4 = reinterpret_cast<const float4*>(ws);
  for (int64_t qb = (int64_t)blockIdx.x * Q; qb < quads; qb += (int64_t)gridDim.x * Q) {
    const int64_t quad = qb + quad_l;
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    if (quad < quads && g < splits) {
      acc = w4[(int64_t)g * quads + quad];
      int s = g + G;
      for (; s + 3 * G < splits; s += 4 * G) {
        const float4 a = w4[(int64_t)s * quads + quad];
        const float4 b = w4[(int64_t)(s + G) * quads + quad];
        const float4 c = w4[(int64_t)(s + 2 * G) * quads + quad];
        const float4 d = w4[(int64_t)(s + 3 * G) * quads + quad];
        acc.x = __fadd_rn(__fadd_rn(__fadd_rn(__fadd_rn(acc.x, a.x), b.x), c.x), d.x);
        acc.y = __fadd_rn(__fadd_rn(__fadd_rn(__fadd_rn(acc.y, a.y), b.y), c.y), d.y);
        acc.z = __fadd_rn(__fadd_rn(__fadd_rn(__fadd_rn(acc.z, a.z), b.z), c.z), d.z);
        acc.w = __fadd_rn(__fadd_rn(__fadd_rn(__fadd_rn(acc.w, a.w), b.w), c.w), d.w);
      }
      for (; s < splits; s += G) {
        const float4 a = w4[(int64_t)s * quads + quad];
        acc.x = __fadd_rn(acc.x, a.x);
        acc.y = __fadd_rn(acc.y, a.y);
        acc.z = __fadd_rn(acc.z, a.z);
        acc.w = __fadd_rn(acc.w, a.w);
      }
    }
    if (G > 1) {
      part[t] = acc;
      __syncthreads();
      if (g == 0)
        for (int q = 1; q < G && q < splits; ++q) {
          const float4 a = part[q * Q + quad_l];
          acc.x = __fadd_rn(acc.x, a.x);
          acc.y = __fadd_rn(acc.y, a.y);
          acc.z = __fadd_rn(acc.z, a.z);
          acc.w = __fadd_rn(acc.w, a.w);
        }
      __syncthreads();
    }
    if (g == 0 && quad < quads) {
      const float v[4] = {acc.x, acc.y, acc.z, acc.w};
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int64_t i = 4 * quad + j;
        const int n = (int)(i / M), m = (int)(i - (int64_t)n * M);
        epi(m, n, v[j]);
      }
    }
  }
}

// launch the split-K reduction that suits the split count
template <class Epi>
inline void splitk_reduce(const float* ws, int splits, int M, int N, const Epi& epi,
                          cudaStream_t st) {
  const int64_t total = (int64_t)M * N;
  if (splits >= 8 && total % 4 == 0 && (reinterpret_cast<uintptr_t>(ws) & 15) == 0) {
    const int64_t quads = total / 4;
    const int64_t want = (int64_t)sm_count_current() * 2048;
    int G = 1;
    while (G < 32 && G < splits && quads * G < want) G *= 2;
    const int Q = 256 / G;
    const int64_t blocks = (quads + Q - 1) / Q;
    const int grid = (int)std::min<int64_t>(blocks, (int64_t)sm_count_current() * 8);
    splitk_reduce_vec_kernel<Epi><<<grid, 256, 0, st>>>(ws, splits, M, N, G, epi);
  } else {
    splitk_reduce_kernel<Epi><<<elementwise_grid(total, 256), 256, 0, st>>>(ws, splits, M, N,
                                                                            epi);
  }
}

// Tensor-core accumulation is not round-to-nearest: tcgen05.mma rounds each
// instruction's fp32 sum toward zero, so a reduction chain of L k-blocks (12
// kind::tf32 MMAs each under 3xTF32) shrinks its result by ~2e-7 * L
// (tools/precision_probe.py; profiles/r02_precision.md).  Weight gradients
// reduce over K = N*P*Q (401k at GoogLeNet's 56x56 layers, batch 128), so
// their K loop is split into chains of at most max_chain_kb() k-blocks whose
// partials are summed in fp32 round-to-nearest by the split-K reduction.
// PURINE_B200_MAX_CHAIN_KB overrides the default of 32 (1024 elements); 0
// disables the bound.
constexpr int kMaxSplits = 4096;
int max_chain_kb();
// sacc: the tile keeps its small terms in a separate accumulator (one
// truncating accumulation of the big part per k-step instead of three), so a
// chain may be three times as long for the same error (precision_probe,
// K = 401k: 32-k-block chains 1.7e-6 of max |ref| with it vs 6.4e-6 without;
// 96-k-block chains 5.1e-6)
int chain_plain_mult();  // PURINE_B200_CHAIN_PLAIN: chain multiplier without the small accumulator
inline int64_t chain_min_splits(int64_t nkb, bool sacc = false) {
  const int c = max_chain_kb() * (sacc ? 3 : chain_plain_mult());
  return c > 0 ? (nkb + c - 1) / c : 1;
}

// Weight-gradient split-K factor: at least s_min (SM fill / chain bound), at
// most s_max (workspace, k-blocks); among those, the fewest k-blocks on the
// busiest CTA of the persistent grid, ceil(units / sms) * (kbps + ramp) with a
// unit's pipeline ramp and epilogue counted as kRamp k-blocks -- so the last
// wave is not a sliver (3a/5x5_reduce: 100 splits = 1.35 waves of 64 k-blocks
// -> 148 splits = 2 waves of 22).  PURINE_B200_BALANCE_SPLITS=0 keeps s_min.
bool balance_splits_enabled();
inline int64_t balance_splits(int64_t tiles, int64_t nkb, int64_t s_min, int64_t s_max,
                              int sms) {
  constexpr int64_t kRamp = 2;
  s_min = std::max<int64_t>(1, s_min);
  s_max = std::max<int64_t>(s_min, s_max);
  if (!balance_splits_enabled() || s_min == 1 && tiles >= sms) return s_min;
  auto cost = [&](int64_t s) {
    const int64_t kbps = (nkb + s - 1) / s;
    const int64_t se = (nkb + kbps - 1) / kbps;
    return ((tiles * se + sms - 1) / sms) * (kbps + kRamp);
  };
  int64_t best = s_min, bc = cost(s_min);
  const int64_t hi = std::min<int64_t>(s_max, 2 * s_min + 8);
  for (int64_t s = s_min + 1; s <= hi; ++s) {
    const int64_t c = cost(s);
    if (c < bc) {
      bc = c;
      best = s;
    }
  }
  return best;
}

enum GemmOp { kConvFwd = 0, kConvDgrad = 1, kConvWgrad = 2, kFcFwd = 3, kFcDgrad = 4, kFcWgrad = 5 };

// choose a split-K factor: fill ~2 waves of SMs, keep >= min_k per split,
// bounded by the workspace
inline int choose_splits(int64_t M, int64_t N, int64_t K, int bm, int bn, int64_t min_k,
                         int64_t ws_bytes) {
  int64_t tiles = ((M + bm - 1) / bm) * ((N + bn - 1) / bn);
  int64_t want = (2LL * gemm_sm_budget() + tiles - 1) / tiles;
  int64_t by_k = K / min_k;
  if (want > by_k) want = by_k;
  if (want > 64) want = 64;
  int64_t by_ws = ws_bytes / (M * N * (int64_t)sizeof(float));
  if (want > by_ws) want = by_ws;
  return want < 1 ? 1 : (int)want;
}

}  // namespace bf
