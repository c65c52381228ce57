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

// relu_forward's arithmetic (ops.py:359-364; elementwise.cu relu1)
__device__ __forceinline__ float relu_value(float v) { return v > 0.f ? v : 0.f; }

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
  __device__ __forceinline__ void operator()(int m, int n, float v) const {
    int img = m / PQ, pq = m - img * PQ;
    if (bias) v = __fadd_rn(v, bias[n]);
    const int64_t o = ((int64_t)img * Cout + n) * PQ + pq;
    if (relu_x) v = relu_x[o] > 0.f ? v : 0.f;
    out[o] = v;
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
    *p = v;
    if (relu_out) p[r.relu_delta] = relu_value(v);
  }
  // 16 consecutive columns of one row (the tcgen05 epilogues): the folded
  // ReLU's x values are all loaded before any store, so the loads overlap
  __device__ __forceinline__ void store16(const RowPtr& r, int n0, const uint32_t (&v)[16],
                                          int nlim) const {
    float m[16];
    if (relu_x) {
      const float* mx = relu_x + (r.p - out) + (int64_t)n0 * PQ;
#pragma unroll
      for (int j = 0; j < 16; ++j) m[j] = j < nlim ? __ldg(mx + (int64_t)j * PQ) : 0.f;
    }
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      if (j >= nlim) continue;
      float x = __uint_as_float(v[j]);
      if (bias) x = __fadd_rn(x, __ldg(bias + n0 + j));
      if (relu_x) x = m[j] > 0.f ? x : 0.f;
      float* p = r.p + (int64_t)(n0 + j) * PQ;
      *p = x;
      if (relu_out) p[r.relu_delta] = relu_value(x);
    }
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
#pragma unroll
    for (int j = 0; j < 16; ++j)
      if (j < nlim) store(r, n0 + j, __uint_as_float(v[j]));
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
