// Elementwise kernels: ReLU, SGD (plain / momentum / lowered mean), rank-ordered
// aggregate, copy, non-finite check.  All HBM-bound: 128-bit vectorised,
// grid-stride, grid sized in multiples of the SM count.  Rounding follows the
// reference exactly (no FMA contraction: every product is rounded before the
// add), so these kernels are bit-identical to the numpy reference.
#include <stdarg.h>
#include <stdlib.h>

#include <algorithm>
#include <atomic>

#include "common.cuh"

namespace bf {

static thread_local char g_err[512];

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

static std::atomic<long long> g_launches{0};

void count_launches(int n) { g_launches.fetch_add(n, std::memory_order_relaxed); }

static std::atomic<int> g_sm_reserve{0};

// SMs the persistent GEMMs leave free for concurrently running collectives
int gemm_sm_budget() {
  const int sms = sm_count_current();
  const int r = g_sm_reserve.load(std::memory_order_relaxed);
  return sms - r >= 1 ? sms - r : 1;
}

int max_chain_kb() {
  static const int v = [] {
    const char* e = getenv("PURINE_B200_MAX_CHAIN_KB");
    return e && *e ? atoi(e) : 32;
  }();
  return v;
}

int chain_plain_mult() {
  static const int v = [] {
    const char* e = getenv("PURINE_B200_CHAIN_PLAIN");
    return e && *e && atoi(e) > 0 ? atoi(e) : 1;
  }();
  return v;
}

// PURINE_B200_RELU_V4K=0: the grid-stride slice kernels instead of the 2-D ones
static bool v4k_enabled() {
  static const bool v = [] {
    const char* e = getenv("PURINE_B200_RELU_V4K");
    return !(e && *e == '0');
  }();
  return v;
}

int sm_count_current() {
  int dev = 0;
  cudaGetDevice(&dev);
  static int cached[64] = {0};
  if (dev < 0 || dev >= 64) return 148;
  if (cached[dev] == 0) {
    int v = 0;
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    cached[dev] = v > 0 ? v : 148;
  }
  return cached[dev];
}

namespace {

constexpr int kThreads = 256;

// numpy maximum(x, 0) on finite x: x when x > 0, else +0.0 (-0.0 -> +0.0)
// np.maximum(x, 0): NaN propagates, -0 -> +0 (ops.py:359-364)
__device__ __forceinline__ float relu1(float x) { return !(x <= 0.f) ? x : 0.f; }
__device__ __forceinline__ float relu_g(float x, float g) { return x > 0.f ? g : 0.f; }
__device__ __forceinline__ float sgd1(float w, float g, float lr) {
  return __fsub_rn(w, __fmul_rn(lr, g));
}

__global__ void relu_fwd_v4(const float4* __restrict__ x, float4* __restrict__ y, int64_t n4) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4;
       i += (int64_t)gridDim.x * blockDim.x) {
    float4 v = x[i];
    y[i] = make_float4(relu1(v.x), relu1(v.y), relu1(v.z), relu1(v.w));
  }
}

__global__ void relu_fwd_s(const float* __restrict__ x, float* __restrict__ y, int64_t lo,
                           int64_t n) {
  for (int64_t i = lo + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    y[i] = relu1(x[i]);
}

__global__ void relu_bwd_v4(const float4* __restrict__ x, const float4* __restrict__ dy,
                            float4* __restrict__ dx, int64_t n4) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4;
       i += (int64_t)gridDim.x * blockDim.x) {
    float4 a = x[i], g = dy[i];
    dx[i] = make_float4(relu_g(a.x, g.x), relu_g(a.y, g.y), relu_g(a.z, g.z), relu_g(a.w, g.w));
  }
}

__global__ void relu_bwd_s(const float* __restrict__ x, const float* __restrict__ dy,
                           float* __restrict__ dx, int64_t lo, int64_t n) {
  for (int64_t i = lo + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    dx[i] = relu_g(x[i], dy[i]);
}

// relu_backward with dy read as a channel slice of a concatenated gradient
// (the graph's concat_backward copy is elided): image n of dx/x covers
// `run` = C*HW contiguous elements, its dy run starts at n*dy_img + dy_off
// x (the ReLU mask) likewise at img*x_img + x_off: the pre-activation itself
// (x_img = run, x_off = 0) or the ReLU output's slice of the concat output
__global__ void relu_bwd_slice_v4(const float4* __restrict__ x, const float4* __restrict__ dy,
                                  float4* __restrict__ dx, int64_t run4, int64_t dy_img4,
                                  int64_t dy_off4, int64_t x_img4, int64_t x_off4, int64_t n4) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t img = i / run4, r = i - img * run4;
    float4 a = x[img * x_img4 + x_off4 + r], g = dy[img * dy_img4 + dy_off4 + r];
    dx[i] = make_float4(relu_g(a.x, g.x), relu_g(a.y, g.y), relu_g(a.z, g.z), relu_g(a.w, g.w));
  }
}

__global__ void relu_bwd_slice_s(const float* __restrict__ x, const float* __restrict__ dy,
                                 float* __restrict__ dx, int64_t run, int64_t dy_img,
                                 int64_t dy_off, int64_t x_img, int64_t x_off, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t img = i / run, r = i - img * run;
    dx[i] = relu_g(x[img * x_img + x_off + r], dy[img * dy_img + dy_off + r]);
  }
}

__global__ void sgd_kernel(const float* __restrict__ w, const float* __restrict__ g,
                           float* __restrict__ out, float lr, int64_t n) {
  int64_t n4 = n >> 2;
  const float4* w4 = reinterpret_cast<const float4*>(w);
  const float4* g4 = reinterpret_cast<const float4*>(g);
  float4* o4 = reinterpret_cast<float4*>(out);
  int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4; i += stride) {
    float4 a = w4[i], b = g4[i];
    o4[i] = make_float4(sgd1(a.x, b.x, lr), sgd1(a.y, b.y, lr), sgd1(a.z, b.z, lr),
                        sgd1(a.w, b.w, lr));
  }
  for (int64_t i = (n4 << 2) + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += stride)
    out[i] = sgd1(w[i], g[i], lr);
}

__global__ void sgd_scalar(const float* __restrict__ w, const float* __restrict__ g,
                           float* __restrict__ out, float lr, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = sgd1(w[i], g[i], lr);
}

// SGD family over float4 lanes (the 4-aligned body) plus a scalar tail.
// One functor per update rule keeps the vector and scalar paths identical.
// The lowered exchange divides the reduce-scattered gradient SUM by f32(k)
// (aggregate mean, ops.py:454-455: a true division, not a reciprocal
// multiply) before the update, so at k = 1 it is bitwise the plain rule.
struct MeanSgd {
  float lr, k;
  __device__ __forceinline__ void operator()(float w, float g, float, float& wn, float&) const {
    wn = __fsub_rn(w, __fmul_rn(lr, __fdiv_rn(g, k)));
  }
};
// Caffe momentum (oracle sgd_momentum): v' = mu*v + lr*g; w' = w - v'
struct MeanMomentum {
  float lr, mu, k;
  __device__ __forceinline__ void operator()(float w, float g, float v, float& wn,
                                             float& vn) const {
    vn = __fadd_rn(__fmul_rn(mu, v), __fmul_rn(lr, __fdiv_rn(g, k)));
    wn = __fsub_rn(w, vn);
  }
};

template <class Rule, bool kVel>
__global__ void sgd_family_kernel(const float* __restrict__ w, const float* __restrict__ g,
                                  const float* __restrict__ v, float* __restrict__ w_new,
                                  float* __restrict__ v_new, int64_t n4, int64_t n, Rule rule) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t t0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  for (int64_t i = t0; i < n4; i += stride) {
    const float4 a = reinterpret_cast<const float4*>(w)[i];
    const float4 b = reinterpret_cast<const float4*>(g)[i];
    float4 c = make_float4(0.f, 0.f, 0.f, 0.f), wn, vn;
    if (kVel) c = reinterpret_cast<const float4*>(v)[i];
    rule(a.x, b.x, c.x, wn.x, vn.x);
    rule(a.y, b.y, c.y, wn.y, vn.y);
    rule(a.z, b.z, c.z, wn.z, vn.z);
    rule(a.w, b.w, c.w, wn.w, vn.w);
    reinterpret_cast<float4*>(w_new)[i] = wn;
    if (kVel) reinterpret_cast<float4*>(v_new)[i] = vn;
  }
  for (int64_t i = 4 * n4 + t0; i < n; i += stride) {
    float wn, vn;
    rule(w[i], g[i], kVel ? v[i] : 0.f, wn, vn);
    w_new[i] = wn;
    if (kVel) v_new[i] = vn;
  }
}

template <class Rule, bool kVel>
int launch_sgd_family(const float* w, const float* g, const float* v, float* w_new, float* v_new,
                      int64_t n, Rule rule, cudaStream_t st, const char* what) {
  if (n <= 0) return 0;
  bool vec = aligned16(w) && aligned16(g) && aligned16(w_new);
  if (kVel) vec = vec && aligned16(v) && aligned16(v_new);
  const int64_t n4 = vec ? n / 4 : 0;
  const int64_t items = n4 + (n - 4 * n4);
  sgd_family_kernel<Rule, kVel><<<elementwise_grid(items, kThreads), kThreads, 0, st>>>(
      w, g, v, w_new, v_new, n4, n, rule);
  return check_launch(what);
}

struct Parts {
  const float* p[32];
};

__global__ void aggregate_v4(Parts parts, int k, float4* __restrict__ out, int64_t n4, int mean) {
  const float fk = (float)k;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4;
       i += (int64_t)gridDim.x * blockDim.x) {
    float4 acc = reinterpret_cast<const float4*>(parts.p[0])[i];
    for (int j = 1; j < k; ++j) {
      const float4 v = reinterpret_cast<const float4*>(parts.p[j])[i];
      acc.x = __fadd_rn(acc.x, v.x);
      acc.y = __fadd_rn(acc.y, v.y);
      acc.z = __fadd_rn(acc.z, v.z);
      acc.w = __fadd_rn(acc.w, v.w);
    }
    if (mean) {
      acc.x = __fdiv_rn(acc.x, fk);
      acc.y = __fdiv_rn(acc.y, fk);
      acc.z = __fdiv_rn(acc.z, fk);
      acc.w = __fdiv_rn(acc.w, fk);
    }
    out[i] = acc;
  }
}

__global__ void aggregate_kernel(Parts parts, int k, float* __restrict__ out, int64_t n,
                                 int mean) {
  float fk = (float)k;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    float acc = parts.p[0][i];
    for (int j = 1; j < k; ++j) acc = __fadd_rn(acc, parts.p[j][i]);
    if (mean) acc = __fdiv_rn(acc, fk);
    out[i] = acc;
  }
}

// device-side injected latency (the reference's delay_s / copy_latency_s,
// dispatcher.py:289-294, ops.py:539-540): occupies the lane's stream
__global__ void delay_kernel(int64_t ns) {
  uint64_t t0, t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  do {
    __nanosleep(1000);
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  } while ((int64_t)(t - t0) < ns);
}

__global__ void finite_kernel(const float* __restrict__ x, int64_t n, int* flag) {
  bool bad = false;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    bad |= !isfinite(x[i]);
  if (__syncthreads_or(bad) && threadIdx.x == 0) *flag = 1;
}

// up to kFiniteMax tensors per launch, passed by value (no device-side table:
// the launch is safe to capture into a CUDA graph and replays with the same
// buffers).  Blocks stride over the concatenation of the tensors; aligned
// tensors are read as float4.
constexpr int kFiniteMax = 96;
struct FiniteList {
  const float* ptr[kFiniteMax];
  int64_t len[kFiniteMax];
  int count;
};

// grid (chunks, tensors): block (x, t) checks chunk x of tensor t (4096
// floats); blocks past a tensor's end exit at once.  (A grid-stride walk over
// the tensors one after another was latency-bound on the ~116 small parameter
// tensors: 38 us per launch for 14 MB.)
constexpr int kFiniteChunk = 4096;
__global__ void finite_list_kernel(const FiniteList list, int* flag) {
  const int t = blockIdx.y;
  const float* x = list.ptr[t];
  const int64_t n = list.len[t];
  const int64_t lo = (int64_t)blockIdx.x * kFiniteChunk;
  if (lo >= n) return;
  const int64_t hi = min(n, lo + kFiniteChunk);
  bool bad = false;
  if ((reinterpret_cast<uintptr_t>(x + lo) & 15) == 0 && hi - lo == kFiniteChunk) {
    const float4* x4 = reinterpret_cast<const float4*>(x + lo);
#pragma unroll
    for (int j = 0; j < kFiniteChunk / 4 / 256; ++j) {
      const float4 v = __ldg(x4 + j * 256 + threadIdx.x);
      bad |= !(isfinite(v.x) && isfinite(v.y) && isfinite(v.z) && isfinite(v.w));
    }
  } else {
    for (int64_t i = lo + threadIdx.x; i < hi; i += blockDim.x) bad |= !isfinite(x[i]);
  }
  if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(flag, 1);
}

// the float4 path for k <= 4 parts: a 2-D grid (blocks over one image's run x
// images) needs no index division, and each thread loads every part's float4
// and the mask's for two elements before summing -- 2 * (K + 1) loads in
// flight instead of one.  Same summation order as relu_bwd_slice_sum_v4: bitwise
// the same.
template <int K>
__global__ void __launch_bounds__(256)
    relu_bwd_slice_sum_v4k(const float4* __restrict__ x, Parts parts, float4* __restrict__ dx,
                           int64_t run4, int64_t dy_img4, int64_t dy_off4, int64_t x_img4,
                           int64_t x_off4) {
  const int64_t img = blockIdx.y;
  const float4* __restrict__ xs = x + img * x_img4 + x_off4;
  float4* __restrict__ d = dx + img * run4;
  const int64_t base = img * dy_img4 + dy_off4;
  const int64_t step = (int64_t)gridDim.x * 2 * blockDim.x;
  for (int64_t r0 = (int64_t)blockIdx.x * 2 * blockDim.x + threadIdx.x; r0 < run4; r0 += step) {
    const int64_t r1 = r0 + blockDim.x;
    const bool h1 = r1 < run4;
    float4 v0[K], v1[K];
#pragma unroll
    for (int q = 0; q < K; ++q) {
      const float4* __restrict__ pq = reinterpret_cast<const float4*>(parts.p[q]) + base;
      v0[q] = pq[r0];
      v1[q] = h1 ? pq[r1] : make_float4(0.f, 0.f, 0.f, 0.f);
    }
    const float4 a0 = xs[r0];
    const float4 a1 = h1 ? xs[r1] : make_float4(0.f, 0.f, 0.f, 0.f);
    float4 g0 = v0[0], g1 = v1[0];
#pragma unroll
    for (int q = 1; q < K; ++q) {
      g0.x = __fadd_rn(g0.x, v0[q].x);
      g0.y = __fadd_rn(g0.y, v0[q].y);
      g0.z = __fadd_rn(g0.z, v0[q].z);
      g0.w = __fadd_rn(g0.w, v0[q].w);
      g1.x = __fadd_rn(g1.x, v1[q].x);
      g1.y = __fadd_rn(g1.y, v1[q].y);
      g1.z = __fadd_rn(g1.z, v1[q].z);
      g1.w = __fadd_rn(g1.w, v1[q].w);
    }
    d[r0] = make_float4(relu_g(a0.x, g0.x), relu_g(a0.y, g0.y), relu_g(a0.z, g0.z),
                        relu_g(a0.w, g0.w));
    if (h1)
      d[r1] = make_float4(relu_g(a1.x, g1.x), relu_g(a1.y, g1.y), relu_g(a1.z, g1.z),
                          relu_g(a1.w, g1.w));
  }
}

// launch relu_bwd_slice_sum_v4k for k in 1..4 parts; false for other k
inline bool launch_slice_sum_v4k(const float4* x, const Parts& p, int k, float4* dx, int N,
                                 int64_t run4, int64_t dy_img4, int64_t dy_off4, int64_t x_img4,
                                 int64_t x_off4, cudaStream_t st) {
  if (k < 1 || k > 4 || N < 1 || N > 65535 || !v4k_enabled()) return false;
  const int64_t per_img = (run4 + 2 * kThreads - 1) / (2 * kThreads);
  const int64_t cap = std::max<int64_t>(1, (int64_t)sm_count_current() * 8 / N);
  const dim3 grid((unsigned)std::min(per_img, cap), (unsigned)N);
  switch (k) {
    case 1:
      relu_bwd_slice_sum_v4k<1><<<grid, kThreads, 0, st>>>(x, p, dx, run4, dy_img4, dy_off4,
                                                            x_img4, x_off4);
      break;
    case 2:
      relu_bwd_slice_sum_v4k<2><<<grid, kThreads, 0, st>>>(x, p, dx, run4, dy_img4, dy_off4,
                                                            x_img4, x_off4);
      break;
    case 3:
      relu_bwd_slice_sum_v4k<3><<<grid, kThreads, 0, st>>>(x, p, dx, run4, dy_img4, dy_off4,
                                                            x_img4, x_off4);
      break;
    default:
      relu_bwd_slice_sum_v4k<4><<<grid, kThreads, 0, st>>>(x, p, dx, run4, dy_img4, dy_off4,
                                                            x_img4, x_off4);
      break;
  }
  return true;
}

}  // namespace
}  // namespace bf

using namespace bf;

extern "C" {

int bf_version(void) { return 1; }

long long bf_launch_count(void) { return bf::g_launches.load(); }

const char* bf_last_error(void) { return bf::g_err; }

int bf_sm_count(int device) {
  int v = 0;
  if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, device) != cudaSuccess) {
    set_error("bf_sm_count: cannot query device %d", device);
    return -1;
  }
  return v;
}

int bf_set_sm_reserve(int n) {
  BF_REQUIRE(n >= 0 && n < sm_count_current(), "bf_set_sm_reserve: 0 <= n < SM count");
  g_sm_reserve.store(n, std::memory_order_relaxed);
  return 0;
}

int bf_set_device(int device) {
  BF_CUDA(cudaSetDevice(device), "bf_set_device");
  return 0;
}

int bf_delay_ns(int64_t ns, bf_stream_t s) {
  if (ns <= 0) return 0;
  delay_kernel<<<1, 1, 0, as_stream(s)>>>(ns);
  return check_launch("delay");
}

int bf_relu_fwd(const float* x, float* y, int64_t n, bf_stream_t s) {
  if (n <= 0) return 0;
  cudaStream_t st = as_stream(s);
  int64_t n4 = aligned16(x) && aligned16(y) ? n / 4 : 0;
  if (n4) relu_fwd_v4<<<elementwise_grid(n4, kThreads), kThreads, 0, st>>>(
      reinterpret_cast<const float4*>(x), reinterpret_cast<float4*>(y), n4);
  if (n4 * 4 < n) relu_fwd_s<<<elementwise_grid(n - n4 * 4, kThreads), kThreads, 0, st>>>(
      x, y, n4 * 4, n);
  return check_launch("relu_forward", (n4 > 0) + (n4 * 4 < n));
}

int bf_relu_bwd(const float* x, const float* dy, float* dx, int64_t n, bf_stream_t s) {
  if (n <= 0) return 0;
  cudaStream_t st = as_stream(s);
  int64_t n4 = aligned16(x) && aligned16(dy) && aligned16(dx) ? n / 4 : 0;
  if (n4) relu_bwd_v4<<<elementwise_grid(n4, kThreads), kThreads, 0, st>>>(
      reinterpret_cast<const float4*>(x), reinterpret_cast<const float4*>(dy),
      reinterpret_cast<float4*>(dx), n4);
  if (n4 * 4 < n) relu_bwd_s<<<elementwise_grid(n - n4 * 4, kThreads), kThreads, 0, st>>>(
      x, dy, dx, n4 * 4, n);
  return check_launch("relu_backward", (n4 > 0) + (n4 * 4 < n));
}

// relu_backward whose dy is the channel slice of a rank-ordered SUM of k
// concatenated gradients: the graph's aggregate(sum) -> concat_backward pair is
// elided (ops.py:440-457 order: ((p0 + p1) + p2) + ...)
__global__ void relu_bwd_slice_sum_v4(const float4* __restrict__ x, Parts parts, int k,
                                      float4* __restrict__ dx, int64_t run4, int64_t dy_img4,
                                      int64_t dy_off4, int64_t x_img4, int64_t x_off4,
                                      int64_t n4) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t img = i / run4, r = i - img * run4;
    const int64_t j = img * dy_img4 + dy_off4 + r;
    float4 g = reinterpret_cast<const float4*>(parts.p[0])[j];
    for (int q = 1; q < k; ++q) {
      const float4 v = reinterpret_cast<const float4*>(parts.p[q])[j];
      g.x = __fadd_rn(g.x, v.x);
      g.y = __fadd_rn(g.y, v.y);
      g.z = __fadd_rn(g.z, v.z);
      g.w = __fadd_rn(g.w, v.w);
    }
    const float4 a = x[img * x_img4 + x_off4 + r];
    dx[i] = make_float4(relu_g(a.x, g.x), relu_g(a.y, g.y), relu_g(a.z, g.z), relu_g(a.w, g.w));
  }
}

__global__ void relu_bwd_slice_sum_s(const float* __restrict__ x, Parts parts, int k,
                                     float* __restrict__ dx, int64_t run, int64_t dy_img,
                                     int64_t dy_off, int64_t x_img, int64_t x_off, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t img = i / run, r = i - img * run;
    const int64_t j = img * dy_img + dy_off + r;
    float g = parts.p[0][j];
    for (int q = 1; q < k; ++q) g = __fadd_rn(g, parts.p[q][j]);
    dx[i] = relu_g(x[img * x_img + x_off + r], g);
  }
}

int bf_relu_bwd_slice_sum_x(const float* x, int x_c0, int x_ctot, const float* const* parts,
                            int k, int c0, int ctot, float* dx, int N, int C, int64_t HW,
                            bf_stream_t s) {
  BF_REQUIRE(k >= 1 && k <= 32, "relu_backward(slice sum): 1 <= k <= 32 parts, got %d", k);
  BF_REQUIRE(N >= 0 && C >= 0 && c0 >= 0 && c0 + C <= ctot, "relu_backward(slice): bad channels");
  BF_REQUIRE(x_c0 >= 0 && x_c0 + C <= x_ctot, "relu_backward(slice): bad mask channels");
  const int64_t run = (int64_t)C * HW, n = run * N;
  if (n <= 0) return 0;
  cudaStream_t st = as_stream(s);
  Parts p;
  // float4 when every image / slice offset is a multiple of 4 elements (the
  // 7x7 planes of inception 5a/5b qualify through channel counts that are)
  bool vec = aligned16(x) && aligned16(dx) && run % 4 == 0 && ((int64_t)ctot * HW) % 4 == 0 &&
             ((int64_t)c0 * HW) % 4 == 0 && ((int64_t)x_ctot * HW) % 4 == 0 &&
             ((int64_t)x_c0 * HW) % 4 == 0;
  for (int i = 0; i < k; ++i) {
    p.p[i] = parts[i];
    vec = vec && aligned16(parts[i]);
  }
  if (vec && launch_slice_sum_v4k(reinterpret_cast<const float4*>(x), p, k,
                                  reinterpret_cast<float4*>(dx), N, run / 4,
                                  (int64_t)ctot * HW / 4, (int64_t)c0 * HW / 4,
                                  (int64_t)x_ctot * HW / 4, (int64_t)x_c0 * HW / 4, st)) {
  } else if (vec)
    relu_bwd_slice_sum_v4<<<elementwise_grid(n / 4, kThreads), kThreads, 0, st>>>(
        reinterpret_cast<const float4*>(x), p, k, reinterpret_cast<float4*>(dx), run / 4,
        (int64_t)ctot * HW / 4, (int64_t)c0 * HW / 4, (int64_t)x_ctot * HW / 4,
        (int64_t)x_c0 * HW / 4, n / 4);
  else
    relu_bwd_slice_sum_s<<<elementwise_grid(n, kThreads), kThreads, 0, st>>>(
        x, p, k, dx, run, (int64_t)ctot * HW, (int64_t)c0 * HW, (int64_t)x_ctot * HW,
        (int64_t)x_c0 * HW, n);
  return check_launch("relu_backward");
}

int bf_relu_bwd_slice_sum(const float* x, const float* const* parts, int k, int c0, int ctot,
                          float* dx, int N, int C, int64_t HW, bf_stream_t s) {
  return bf_relu_bwd_slice_sum_x(x, 0, C, parts, k, c0, ctot, dx, N, C, HW, s);
}

int bf_relu_bwd_slice_x(const float* x, int x_c0, int x_ctot, const float* dy_cat, int c0,
                        int ctot, float* dx, int N, int C, int64_t HW, bf_stream_t s) {
  BF_REQUIRE(N >= 0 && C >= 0 && c0 >= 0 && c0 + C <= ctot, "relu_backward(slice): bad channels");
  BF_REQUIRE(x_c0 >= 0 && x_c0 + C <= x_ctot, "relu_backward(slice): bad mask channels");
  const int64_t run = (int64_t)C * HW, n = run * N;
  if (n <= 0) return 0;
  cudaStream_t st = as_stream(s);
  if (aligned16(x) && aligned16(dy_cat) && aligned16(dx) && run % 4 == 0 &&
      ((int64_t)ctot * HW) % 4 == 0 && ((int64_t)c0 * HW) % 4 == 0 &&
      ((int64_t)x_ctot * HW) % 4 == 0 && ((int64_t)x_c0 * HW) % 4 == 0) {
    Parts p;
    p.p[0] = dy_cat;
    if (!launch_slice_sum_v4k(reinterpret_cast<const float4*>(x), p, 1,
                              reinterpret_cast<float4*>(dx), N, run / 4, (int64_t)ctot * HW / 4,
                              (int64_t)c0 * HW / 4, (int64_t)x_ctot * HW / 4,
                              (int64_t)x_c0 * HW / 4, st)) {
      relu_bwd_slice_v4<<<elementwise_grid(n / 4, kThreads), kThreads, 0, st>>>(
          reinterpret_cast<const float4*>(x), reinterpret_cast<const float4*>(dy_cat),
          reinterpret_cast<float4*>(dx), run / 4, (int64_t)ctot * HW / 4, (int64_t)c0 * HW / 4,
          (int64_t)x_ctot * HW / 4, (int64_t)x_c0 * HW / 4, n / 4);
    }
  } else {
    relu_bwd_slice_s<<<elementwise_grid(n, kThreads), kThreads, 0, st>>>(
        x, dy_cat, dx, run, (int64_t)ctot * HW, (int64_t)c0 * HW, (int64_t)x_ctot * HW,
        (int64_t)x_c0 * HW, n);
  }
  return check_launch("relu_backward");
}

int bf_relu_bwd_slice(const float* x, const float* dy_cat, int c0, int ctot, float* dx, int N,
                      int C, int64_t HW, bf_stream_t s) {
  return bf_relu_bwd_slice_x(x, 0, C, dy_cat, c0, ctot, dx, N, C, HW, s);
}

int bf_sgd_update(const float* w, const float* g, float* out, float lr, int64_t n,
                  bf_stream_t s) {
  if (n <= 0) return 0;
  if (aligned16(w) && aligned16(g) && aligned16(out))
    sgd_kernel<<<elementwise_grid((n + 3) / 4, kThreads), kThreads, 0, as_stream(s)>>>(
        w, g, out, lr, n);
  else
    sgd_scalar<<<elementwise_grid(n, kThreads), kThreads, 0, as_stream(s)>>>(w, g, out, lr, n);
  return check_launch("sgd_update");
}

int bf_sgd_momentum(const float* w, const float* g, const float* v, float* w_new, float* v_new,
                    float lr, float momentum, int64_t n, bf_stream_t s) {
  return launch_sgd_family<MeanMomentum, true>(w, g, v, w_new, v_new, n,
                                               MeanMomentum{lr, momentum, 1.f}, as_stream(s),
                                               "sgd_momentum");
}

int bf_sgd_mean_update(const float* w, const float* gsum, float* out, float lr, int k,
                       int64_t n, bf_stream_t s) {
  BF_REQUIRE(k >= 1, "sgd_mean_update: k must be >= 1");
  return launch_sgd_family<MeanSgd, false>(w, gsum, nullptr, out, nullptr, n,
                                           MeanSgd{lr, (float)k}, as_stream(s),
                                           "sgd_mean_update");
}

int bf_sgd_mean_momentum(const float* w, const float* gsum, const float* v, float* w_new,
                         float* v_new, float lr, float momentum, int k, int64_t n,
                         bf_stream_t s) {
  BF_REQUIRE(k >= 1, "sgd_mean_momentum: k must be >= 1");
  return launch_sgd_family<MeanMomentum, true>(w, gsum, v, w_new, v_new, n,
                                               MeanMomentum{lr, momentum, (float)k},
                                               as_stream(s), "sgd_mean_momentum");
}

int bf_aggregate(const float* const* parts, int k, float* out, int64_t n, int mean,
                 bf_stream_t s) {
  BF_REQUIRE(k >= 1 && k <= 32, "aggregate: 1 <= k <= 32 inputs supported, got %d", k);
  if (n <= 0) return 0;
  Parts p;
  bool vec = aligned16(out) && n % 4 == 0;
  for (int i = 0; i < k; ++i) {
    p.p[i] = parts[i];
    vec = vec && aligned16(parts[i]);
  }
  if (vec)
    aggregate_v4<<<elementwise_grid(n / 4, kThreads), kThreads, 0, as_stream(s)>>>(
        p, k, reinterpret_cast<float4*>(out), n / 4, mean);
  else
    aggregate_kernel<<<elementwise_grid(n, kThreads), kThreads, 0, as_stream(s)>>>(p, k, out, n,
                                                                                   mean);
  return check_launch("aggregate");
}

int bf_copy(float* dst, int dst_device, const float* src, int src_device, int64_t n,
            bf_stream_t s) {
  if (n <= 0) return 0;
  size_t bytes = (size_t)n * sizeof(float);
  if (dst_device == src_device)
    BF_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToDevice, as_stream(s)), "copy");
  else
    BF_CUDA(cudaMemcpyPeerAsync(dst, dst_device, src, src_device, bytes, as_stream(s)),
            "copy(peer)");
  return 0;
}

int bf_check_finite(const float* x, int64_t n, int* flag, bf_stream_t s) {
  if (n <= 0) return 0;
  finite_kernel<<<elementwise_grid(n, kThreads), kThreads, 0, as_stream(s)>>>(x, n, flag);
  return check_launch("check_finite");
}

int bf_check_finite_list(const float* const* ptrs, const int64_t* lens, int count, int* flag,
                         bf_stream_t s) {
  if (count < 0 || (count > 0 && (!ptrs || !lens || !flag))) {
    set_error("check_finite_list: bad arguments (count %d)", count);
    return -1;
  }
  for (int base = 0; base < count; base += kFiniteMax) {
    FiniteList list;
    list.count = count - base < kFiniteMax ? count - base : kFiniteMax;
    int64_t longest = 0;
    for (int i = 0; i < list.count; ++i) {
      list.ptr[i] = ptrs[base + i];
      list.len[i] = lens[base + i];
      longest = std::max<int64_t>(longest, lens[base + i]);
    }
    if (longest <= 0) continue;
    const dim3 grid((unsigned)((longest + kFiniteChunk - 1) / kFiniteChunk), (unsigned)list.count);
    finite_list_kernel<<<grid, 256, 0, as_stream(s)>>>(list, flag);
    const int rc = check_launch("check_finite_list");
    if (rc) return rc;
  }
  return 0;
}

}  // extern "C"
