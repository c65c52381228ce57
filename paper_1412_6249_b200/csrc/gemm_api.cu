// C-ABI entry points for the dense contractions: conv fwd / dgrad / wgrad and
// the fully connected layer (reference ops.py:164-343).  Each maps its
// operator onto D[m][n] = sum_k A(m,k) B(n,k) (gemm_common.cuh) and hands it
// to the tcgen05 engine, or the SIMT engine when the tcgen05 engine declines
// the shape or SIMT is forced.
#include "gemm_common.cuh"
#include "gemm_engines.cuh"

namespace bf {

int g_gemm_engine = 0;

template <class LA, class LB, class Epi>
static int run_gemm(const LA& la, const LB& lb, int M, int N, int K, const Epi& epi, float* ws,
                    int64_t ws_bytes, cudaStream_t st, const char* what) {
  if (g_gemm_engine != 1) {
    int rc = tc_gemm(la, lb, M, N, K, epi, ws, ws_bytes, st, what);
    if (rc >= 0) return rc;
  }
  return simt_gemm(la, lb, M, N, K, epi, ws, ws_bytes, st, what);
}

static int check_conv(int N, int C, int H, int W, int K, int R, int S, int P, int Q, int stride,
                      int pad) {
  BF_REQUIRE(N > 0 && C > 0 && H > 0 && W > 0 && K > 0 && R > 0 && S > 0 && P > 0 && Q > 0,
             "conv2d: non-positive dimension");
  BF_REQUIRE(stride >= 1 && pad >= 0, "conv2d: bad stride/pad");
  BF_REQUIRE((H + 2 * pad - R) / stride + 1 == P && (W + 2 * pad - S) / stride + 1 == Q,
             "conv2d: output dims %dx%d do not match geometry", P, Q);
  BF_REQUIRE((int64_t)N * C * H * W < (1LL << 31) && (int64_t)N * K * P * Q < (1LL << 31),
             "conv2d: tensor too large for 32-bit pixel indexing");
  return 0;
}

}  // namespace bf

using namespace bf;

extern "C" {

int bf_set_gemm_engine(int engine) {
  BF_REQUIRE(engine >= 0 && engine <= 7,
             "bf_set_gemm_engine: 0 (auto), 1 (simt), 2 (tcgen05 v1 only), 3 (auto + halo engine "
             "v3), 4 (auto without the 1x1 TMA engine v4), 5 (auto without the TMA-fed 1x1 "
             "weight gradient), 6 (auto with register-prefetched gathers), 7 (auto + TMA-streamed "
             "raw dY for conv1-type weight gradients)");
  g_gemm_engine = engine;
  return 0;
}

int bf_conv2d_fwd(const float* x, const float* w, const float* b, float* y, int N, int C, int H,
                  int W, int K, int R, int S, int P, int Q, int stride, int pad, float* ws,
                  int64_t ws_bytes, bf_stream_t s) {
  return bf_conv2d_fwd_relu(x, w, b, y, nullptr, N, C, H, W, K, R, S, P, Q, stride, pad, ws,
                            ws_bytes, s);
}

int bf_conv2d_fwd_relu(const float* x, const float* w, const float* b, float* y, float* y_relu,
                       int N, int C, int H, int W, int K, int R, int S, int P, int Q, int stride,
                       int pad, float* ws, int64_t ws_bytes, bf_stream_t s) {
  return bf_conv2d_fwd_relu_slice(x, w, b, y, y_relu, 0, K, N, C, H, W, K, R, S, P, Q, stride,
                                  pad, ws, ws_bytes, s);
}

int bf_conv2d_fwd_relu_slice(const float* x, const float* w, const float* b, float* y,
                             float* relu_cat, int relu_c0, int relu_ctot, int N, int C, int H,
                             int W, int K, int R, int S, int P, int Q, int stride, int pad,
                             float* ws, int64_t ws_bytes, bf_stream_t s) {
  if (int rc = check_conv(N, C, H, W, K, R, S, P, Q, stride, pad)) return rc;
  BF_REQUIRE(!relu_cat || (relu_c0 >= 0 && relu_c0 + K <= relu_ctot),
             "conv2d_forward(+relu slice): bad channel range");
  BF_REQUIRE(y || relu_cat, "conv2d_forward: no output (y and the ReLU target are both NULL)");
  ConvShape g{N, C, H, W, K, R, S, P, Q, stride, pad};
  LdFwdX la{x, g};
  LdRowK lb{w, (int64_t)C * R * S};
  EpiNCHW epi{y, b, P * Q, K, relu_cat, (int64_t)relu_ctot * P * Q, relu_c0};
  epi.no_out = y == nullptr;  // pre-activation not stored: only the ReLU output
  if (g_gemm_engine == 0 || g_gemm_engine == 5 || g_gemm_engine == 6 || g_gemm_engine == 7 || g_gemm_engine == 3) {
    int rc = tc4_conv_fwd(g, x, w, epi, ws, ws_bytes, as_stream(s), "conv2d_forward");
    if (rc >= 0) return rc;
  }
  if (g_gemm_engine == 0 && C * R * S <= 256 && K <= 64 && !s2d_enabled()) {
    int rc = fwd_win_conv(g, x, w, epi, ws, ws_bytes, as_stream(s), "conv2d_forward");
    if (rc >= 0) return rc;
  }
  if (g_gemm_engine == 0) {
    int rc = s2d_conv_fwd(g, x, w, epi, ws, ws_bytes, as_stream(s), "conv2d_forward");
    if (rc >= 0) return rc;
  }
  if (g_gemm_engine == 3) {
    int rc = tc3_conv_fwd(g, x, w, epi, ws, ws_bytes, as_stream(s), "conv2d_forward");
    if (rc >= 0) return rc;
  }
  if (g_gemm_engine == 0 || g_gemm_engine == 5 || g_gemm_engine == 6 || g_gemm_engine == 7 || g_gemm_engine == 3 || g_gemm_engine == 4) {
    int rc = tc2_conv_fwd(la, lb, N * P * Q, K, C * R * S, epi, ws, ws_bytes, as_stream(s),
                          "conv2d_forward");
    if (rc >= 0) return rc;
  }
  return run_gemm(la, lb, N * P * Q, K, C * R * S, epi, ws, ws_bytes, as_stream(s),
                  "conv2d_forward");
}

int bf_conv1x1_fwd_group(const float* x, int N, int C, int H, int W, int nseg,
                         const float* const* w, const float* const* b, const int* kout,
                         float* const* y, float* const* relu, const int* relu_c0,
                         const int* relu_ctot, float* ws, int64_t ws_bytes, bf_stream_t s) {
  BF_REQUIRE(nseg >= 1 && nseg <= kMaxSeg, "conv1x1 group: 1 <= nseg <= %d, got %d", kMaxSeg,
             nseg);
  BF_REQUIRE(N > 0 && C > 0 && H > 0 && W > 0, "conv1x1 group: non-positive dimension");
  EpiNCHWSeg epi{};
  epi.PQ = H * W;
  epi.nseg = nseg;
  int n = 0;
  for (int i = 0; i < nseg; ++i) {
    BF_REQUIRE(kout[i] > 0 && w[i] && (y[i] || relu[i]), "conv1x1 group: segment %d malformed",
               i);
    BF_REQUIRE(!relu[i] || (relu_c0[i] >= 0 && relu_c0[i] + kout[i] <= relu_ctot[i]),
               "conv1x1 group: segment %d relu channel range", i);
    epi.start[i] = n;
    epi.out[i] = y[i];
    epi.bias[i] = b[i];
    epi.cout[i] = kout[i];
    epi.relu[i] = relu[i];
    epi.relu_img[i] = relu[i] ? (int64_t)relu_ctot[i] * H * W : 0;
    epi.relu_c0[i] = relu[i] ? relu_c0[i] : 0;
    n += kout[i];
  }
  for (int i = nseg; i <= kMaxSeg; ++i) epi.start[i] = n;
  BF_REQUIRE((int64_t)N * C * H * W < (1LL << 31) && (int64_t)N * n * H * W < (1LL << 31),
             "conv1x1 group: tensor too large for 32-bit pixel indexing");
  const int rc = tc4_conv_fwd_group(x, N, C, H * W, nseg, w, kout, epi, ws, ws_bytes,
                                    as_stream(s), "conv2d_forward(group)");
  BF_REQUIRE(rc >= 0, "conv1x1 group: shape not taken by the TMA-fed 1x1 engine");
  return rc;
}

int bf_conv1x1_dgrad_group(int N, int C, int H, int W, int nseg, const float* const* dy,
                           const float* const* w, const int* kout, float* dx, float* ws,
                           int64_t ws_bytes, bf_stream_t s) {
  BF_REQUIRE(nseg >= 1 && nseg <= kMaxSeg, "conv1x1 dgrad group: 1 <= nseg <= %d, got %d",
             kMaxSeg, nseg);
  BF_REQUIRE(N > 0 && C > 0 && H > 0 && W > 0, "conv1x1 dgrad group: non-positive dimension");
  for (int i = 0; i < nseg; ++i)
    BF_REQUIRE(kout[i] > 0 && dy[i] && w[i], "conv1x1 dgrad group: segment %d malformed", i);
  BF_REQUIRE((int64_t)N * C * H * W < (1LL << 31), "conv1x1 dgrad group: tensor too large");
  EpiNCHW epi{dx, nullptr, H * W, C};
  const int rc = tc4_conv_dgrad_group(N, C, H * W, nseg, dy, w, kout, epi, ws, ws_bytes,
                                      as_stream(s), "conv2d_backward_data(group)");
  BF_REQUIRE(rc >= 0, "conv1x1 dgrad group: shape not taken by the TMA-fed 1x1 engine");
  return rc;
}

int bf_conv2d_bwd_data(const float* w, const float* dy, float* dx, int N, int C, int H, int W,
                       int K, int R, int S, int P, int Q, int stride, int pad, float* ws,
                       int64_t ws_bytes, bf_stream_t s) {
  return bf_conv2d_bwd_data_relu(w, dy, dx, nullptr, N, C, H, W, K, R, S, P, Q, stride, pad, ws,
                                 ws_bytes, s);
}

int bf_conv2d_bwd_data_relu(const float* w, const float* dy, float* dx, const float* relu_x,
                            int N, int C, int H, int W, int K, int R, int S, int P, int Q,
                            int stride, int pad, float* ws, int64_t ws_bytes, bf_stream_t s) {
  if (int rc = check_conv(N, C, H, W, K, R, S, P, Q, stride, pad)) return rc;
  ConvShape g{N, C, H, W, K, R, S, P, Q, stride, pad};
  LdDgradDY la{dy, g};
  LdDgradW lb{w, g};
  EpiNCHW epi{dx, nullptr, H * W, C};
  epi.relu_x = relu_x;
  if (g_gemm_engine == 0 || g_gemm_engine == 5 || g_gemm_engine == 6 || g_gemm_engine == 7 || g_gemm_engine == 3) {
    int rc = tc4_conv_dgrad(g, dy, w, epi, ws, ws_bytes, as_stream(s), "conv2d_backward_data");
    if (rc >= 0) return rc;
  }
  if (g_gemm_engine == 3) {
    int rc = tc3_conv_dgrad(g, dy, w, epi, ws, ws_bytes, as_stream(s), "conv2d_backward_data");
    if (rc >= 0) return rc;
  }
  if (g_gemm_engine == 0 || g_gemm_engine == 5 || g_gemm_engine == 6 || g_gemm_engine == 7 || g_gemm_engine == 3 || g_gemm_engine == 4) {
    int rc = tc2_conv_dgrad(la, lb, N * H * W, C, K * R * S, epi, ws, ws_bytes, as_stream(s),
                            "conv2d_backward_data");
    if (rc >= 0) return rc;
  }
  return run_gemm(la, lb, N * H * W, C, K * R * S, epi, ws, ws_bytes, as_stream(s),
                  "conv2d_backward_data");
}

int bf_conv2d_bwd_weight(const float* x, const float* dy, float* dw, int N, int C, int H, int W,
                         int K, int R, int S, int P, int Q, int stride, int pad, float* ws,
                         int64_t ws_bytes, bf_stream_t s) {
  return bf_conv2d_bwd_weight_bias(x, dy, dw, nullptr, N, C, H, W, K, R, S, P, Q, stride, pad,
                                   ws, ws_bytes, s);
}

int bf_conv2d_bwd_weight_bias(const float* x, const float* dy, float* dw, float* db, int N,
                              int C, int H, int W, int K, int R, int S, int P, int Q, int stride,
                              int pad, float* ws, int64_t ws_bytes, bf_stream_t s) {
  if (int rc = check_conv(N, C, H, W, K, R, S, P, Q, stride, pad)) return rc;
  ConvShape g{N, C, H, W, K, R, S, P, Q, stride, pad};
  LdWgradX la{x, g};
  LdWgradDY lb{dy, g};
  EpiT epi{dw, nullptr, (int64_t)C * R * S};
  int rc = -1;
  bool db_done = false;
  if (g_gemm_engine == 0 && C * R * S <= 256 && stride >= 2)
    rc = wgrad_t_conv(g, x, dy, dw, db, &db_done, ws, ws_bytes, as_stream(s),
                      "conv2d_backward_weight");
  if (rc < 0 && g_gemm_engine == 0)
    rc = s2d_conv_wgrad(g, x, dy, dw, db, &db_done, ws, ws_bytes, as_stream(s),
                        "conv2d_backward_weight");
  if (rc < 0 && (g_gemm_engine == 0 || g_gemm_engine == 5 || g_gemm_engine == 6 || g_gemm_engine == 7 || g_gemm_engine == 3 || g_gemm_engine == 4))
    rc = tc2_conv_wgrad(la, lb, C * R * S, K, N * P * Q, epi, ws, ws_bytes, as_stream(s),
                        "conv2d_backward_weight", db, &db_done);
  if (rc < 0)
    rc = run_gemm(la, lb, C * R * S, K, N * P * Q, epi, ws, ws_bytes, as_stream(s),
                  "conv2d_backward_weight");
  if (rc != 0 || !db || db_done) return rc;
  return bf_conv2d_bwd_bias(dy, db, N, K, P * Q, ws, ws_bytes, s);
}

int bf_fc_fwd(const float* x, const float* w, const float* b, float* y, int n, int d, int m,
              float* ws, int64_t ws_bytes, bf_stream_t s) {
  BF_REQUIRE(n > 0 && d > 0 && m > 0, "fc_forward: non-positive dimension");
  LdColK la{w, m};
  LdRowK lb{x, d};
  EpiT epi{y, b, m};
  return run_gemm(la, lb, m, n, d, epi, ws, ws_bytes, as_stream(s), "fc_forward");
}

int bf_fc_bwd_data(const float* w, const float* dy, float* dx, int n, int d, int m, float* ws,
                   int64_t ws_bytes, bf_stream_t s) {
  BF_REQUIRE(n > 0 && d > 0 && m > 0, "fc_backward_data: non-positive dimension");
  LdRowK la{w, m};
  LdRowK lb{dy, m};
  EpiT epi{dx, nullptr, d};
  return run_gemm(la, lb, d, n, m, epi, ws, ws_bytes, as_stream(s), "fc_backward_data");
}

int bf_fc_bwd_weight(const float* x, const float* dy, float* dw, int n, int d, int m, float* ws,
                     int64_t ws_bytes, bf_stream_t s) {
  BF_REQUIRE(n > 0 && d > 0 && m > 0, "fc_backward_weight: non-positive dimension");
  LdColK la{dy, m};
  LdColK lb{x, d};
  EpiT epi{dw, nullptr, m};
  return run_gemm(la, lb, m, d, n, epi, ws, ws_bytes, as_stream(s), "fc_backward_weight");
}

int64_t bf_gemm_workspace_bytes(int op, int N, int C, int H, int W, int K, int R, int S, int P,
                                int Q, int stride, int pad) {
  (void)op; (void)N; (void)C; (void)H; (void)W; (void)K; (void)R; (void)S; (void)P; (void)Q;
  (void)stride; (void)pad;
  return 64LL << 20;  // one fixed 64 MiB split-K workspace per lane
}

}  // extern "C"
