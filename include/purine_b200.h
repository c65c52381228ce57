/*
 * purine_b200.h — C ABI of the B200 (sm_100a) kernel library for the Purine
 * data-parallel SGD hot path.
 *
 * Every entry point replaces the arithmetic of one reference operator kind:
 * the reference executes each kind through `OpKindSpec.execute` ->
 * `_plain(fn)` -> a numpy kernel (pkg/src/biflow/ops.py:526-533, registry
 * :750-809).  The Python host layer (paper_1412_6249_b200/gpu_ops.py) keeps
 * that plugin interface and calls these functions through ctypes; the
 * binding a maintainer would add to the reference itself is in
 * INTEGRATION.md.
 *
 * Conventions (all entry points):
 *   - plain device pointers, element counts and dims; fp32 row-major NCHW /
 *     KCRS exactly as the reference stores them (ops.py:1-10);
 *   - `stream` is a cudaStream_t (passed as an opaque pointer);
 *   - no allocation, no host synchronisation: work is only enqueued;
 *     temporary storage comes from a caller-provided workspace;
 *   - reentrant and callable from any host thread;
 *   - return 0 on success, non-zero on failure with a message available
 *     from bf_last_error() (thread-local).  The Python shim maps a failure
 *     to KernelError (ops.py:48-49), which the dispatcher turns into
 *     DispatchError (dispatcher.py:296-311).
 *   - integer index outputs (max-pool argmax) are stored as exactly
 *     representable float32 values, matching the reference's all-float32
 *     tensor store (ops.py:79-157).
 */
#ifndef PURINE_B200_H
#define PURINE_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st* bf_stream_t;

/* library identity / errors --------------------------------------------- */
int bf_version(void);
const char* bf_last_error(void);
/* number of SMs of `device` (grid sizing is done in multiples of it) */
int bf_sm_count(int device);
/* leave n SMs free of persistent GEMM CTAs (for NCCL kernels overlapping the
   backward pass; exchange.py sets it when a communicator exists) */
int bf_set_sm_reserve(int n);
/* 1 if the library was compiled with the tcgen05 GEMM path */
int bf_has_tcgen05(void);
/* total kernels launched by this library so far (process-wide counter) */
long long bf_launch_count(void);
/* select the GEMM engine: 0 = auto (tcgen05 v2 > v1 where supported), 1 = SIMT fp32,
   2 = tcgen05 v1 only, 3 = auto with the halo-staged engine v3 for stride-1 R x S convs
   (opt-in: measured slower than v2 on GoogLeNet shapes), 4 = auto without the
   TMA-fed 1x1 engine v4, 5 = auto without the TMA-fed 1x1 weight gradient,
   6 = auto with engine v2's gathers prefetched one k-block ahead in registers
   instead of staged several k-blocks ahead by cp.async, 7 = auto + the raw dY
   streamed by TMA (no dY pack) for weight gradients over 16-aligned pixel
   rows such as conv1's (opt-in: measured neutral) (A/B comparisons) */
int bf_set_gemm_engine(int engine);

/* bind this library's CUDA runtime to `device` for the calling thread */
int bf_set_device(int device);
/* device-side injected latency on `stream` (reference delay_s / copy_latency_s,
   dispatcher.py:289-294, ops.py:539-540) */
int bf_delay_ns(int64_t ns, bf_stream_t stream);

/* elementwise ------------------------------------------------------------ */
/* relu_forward, ops.py:359-364 */
int bf_relu_fwd(const float* x, float* y, int64_t n, bf_stream_t stream);
/* relu_backward, ops.py:367-376 (dy where x > 0) */
int bf_relu_bwd(const float* x, const float* dy, float* dx, int64_t n, bf_stream_t stream);
/* relu_backward with dy = channels [c0, c0 + C) of a concatenated [N][ctot][HW]
   gradient (the concat_backward copy is elided); x, dx are [N][C][HW] */
int bf_relu_bwd_slice(const float* x, const float* dy_cat, int c0, int ctot, float* dx, int N,
                      int C, int64_t HW, bf_stream_t stream);
/* the same with dy = channels [c0, c0 + C) of the rank-ordered sum of k
   concatenated gradients (parts: HOST array of k <= 32 device pointers): the
   aggregate(sum) -> concat_backward pair is elided */
int bf_relu_bwd_slice_sum(const float* x, const float* const* parts, int k, int c0, int ctot,
                          float* dx, int N, int C, int64_t HW, bf_stream_t stream);
/* the two above with the mask x itself a channel slice [x_c0, x_c0 + C) of an
   x_ctot-channel tensor: the ReLU OUTPUT's slice of the (elided-concat)
   concat output, relu(a) > 0 <=> a > 0 -- the pre-activation is then never
   stored (dispatcher pre-activation elision) */
int bf_relu_bwd_slice_x(const float* x, int x_c0, int x_ctot, const float* dy_cat, int c0,
                        int ctot, float* dx, int N, int C, int64_t HW, bf_stream_t stream);
int bf_relu_bwd_slice_sum_x(const float* x, int x_c0, int x_ctot, const float* const* parts,
                            int k, int c0, int ctot, float* dx, int N, int C, int64_t HW,
                            bf_stream_t stream);
/* sgd_update, ops.py:428-437: out = w - f32(lr)*g, product rounded first */
int bf_sgd_update(const float* w, const float* g, float* out, float lr, int64_t n,
                  bf_stream_t stream);
/* sgd_momentum (extension): v' = mu*v + lr*g; w' = w - v' */
int bf_sgd_momentum(const float* w, const float* g, const float* v, float* w_new,
                    float* v_new, float lr, float momentum, int64_t n, bf_stream_t stream);
/* lowered aggregate(mean)+sgd_update (builders.py:589-603): out = w - f32(lr)*(gsum/f32(k)) */
int bf_sgd_mean_update(const float* w, const float* gsum, float* out, float lr, int k,
                       int64_t n, bf_stream_t stream);
/* lowered aggregate(mean)+sgd_momentum on one shard of the exchange (builders.py:
   581-611 with the momentum extension): v' = mu*v + lr*(gsum/f32(k)); w' = w - v' */
int bf_sgd_mean_momentum(const float* w, const float* gsum, const float* v, float* w_new,
                         float* v_new, float lr, float momentum, int k, int64_t n,
                         bf_stream_t stream);
/* aggregate, ops.py:440-457: rank-ordered sum of k parts (k <= 32); mean divides by f32(k) */
int bf_aggregate(const float* const* parts, int k, float* out, int64_t n, int mean,
                 bf_stream_t stream);
/* copy, ops.py:536-541: device-to-device (peer when devices differ) */
int bf_copy(float* dst, int dst_device, const float* src, int src_device, int64_t n,
            bf_stream_t stream);
/* sets *flag (device int) to 1 if any element is non-finite (ops.py:61-64) */
int bf_check_finite(const float* x, int64_t n, int* flag, bf_stream_t stream);
/* the same over `count` tensors in one pass (host arrays of device pointers and
   lengths, copied into the launch: capture-safe); the flag is sticky (atomic OR).
   The dispatcher runs it once per graph over the graph's sink tensors (the loss
   and the updated parameters), the device form of ops.py:61-64's per-kernel check */
int bf_check_finite_list(const float* const* ptrs, const int64_t* lens, int count, int* flag,
                         bf_stream_t stream);

/* softmax cross-entropy, ops.py:394-425 ---------------------------------- */
/* workspace: >= n floats */
int bf_softmax_xent(const float* logits, const float* labels, float* loss, float* dlogits,
                    int n, int k, float* workspace, bf_stream_t stream);

/* dense layer, ops.py:164-226 -------------------------------------------- */
int bf_fc_fwd(const float* x, const float* w, const float* b, float* y, int n, int d, int m,
              float* workspace, int64_t ws_bytes, bf_stream_t stream);
int bf_fc_bwd_data(const float* w, const float* dy, float* dx, int n, int d, int m,
                   float* workspace, int64_t ws_bytes, bf_stream_t stream);
int bf_fc_bwd_weight(const float* x, const float* dy, float* dw, int n, int d, int m,
                     float* workspace, int64_t ws_bytes, bf_stream_t stream);
int bf_fc_bwd_bias(const float* dy, float* db, int n, int m, bf_stream_t stream);

/* convolution, ops.py:229-352 (NCHW x, KCRS w; P,Q = output dims) -------- */
int bf_conv2d_fwd(const float* x, const float* w, const float* b, float* y,
                  int N, int C, int H, int W, int K, int R, int S, int P, int Q,
                  int stride, int pad, float* workspace, int64_t ws_bytes, bf_stream_t stream);
/* conv2d_forward followed by relu_forward (ops.py:359-364) in one kernel:
   writes the pre-activation y and relu(y).  y may be NULL (the dispatcher's
   pre-activation elision: nothing reads y, every relu_backward of this ReLU
   takes relu(y) as its mask): only relu(y) is written */
int bf_conv2d_fwd_relu(const float* x, const float* w, const float* b, float* y, float* y_relu,
                       int N, int C, int H, int W, int K, int R, int S, int P, int Q,
                       int stride, int pad, float* workspace, int64_t ws_bytes,
                       bf_stream_t stream);
/* the same with relu(y) written into channels [relu_c0, relu_c0 + K) of a
   [N][relu_ctot][P][Q] tensor: the graph's following concat_forward copy
   (ops: concat) is elided */
int bf_conv2d_fwd_relu_slice(const float* x, const float* w, const float* b, float* y,
                             float* relu_cat, int relu_c0, int relu_ctot,
                             int N, int C, int H, int W, int K, int R, int S, int P, int Q,
                             int stride, int pad, float* workspace, int64_t ws_bytes,
                             bf_stream_t stream);
int bf_conv2d_bwd_data(const float* w, const float* dy, float* dx,
                       int N, int C, int H, int W, int K, int R, int S, int P, int Q,
                       int stride, int pad, float* workspace, int64_t ws_bytes,
                       bf_stream_t stream);
/* data gradient with relu_backward folded into the epilogue (relu_x laid out as dx) */
int bf_conv2d_bwd_data_relu(const float* w, const float* dy, float* dx, const float* relu_x,
                            int N, int C, int H, int W, int K, int R, int S, int P, int Q,
                            int stride, int pad, float* workspace, int64_t ws_bytes,
                            bf_stream_t stream);
int bf_conv2d_bwd_weight(const float* x, const float* dy, float* dw,
                         int N, int C, int H, int W, int K, int R, int S, int P, int Q,
                         int stride, int pad, float* workspace, int64_t ws_bytes,
                         bf_stream_t stream);
/* conv2d_backward_weight + conv2d_backward_bias on the same dy (ops.py:332-352): the
   bias sums are taken from the weight gradient's dY pass (no second read of dy);
   db may be NULL */
int bf_conv2d_bwd_weight_bias(const float* x, const float* dy, float* dw, float* db,
                              int N, int C, int H, int W, int K, int R, int S, int P, int Q,
                              int stride, int pad, float* workspace, int64_t ws_bytes,
                              bf_stream_t stream);
/* db[k] = sum over (n, p, q) of dy, deterministic order; workspace >= 4*K*slices bytes
   (optional: NULL falls back to one CTA per channel) */
int bf_conv2d_bwd_bias(const float* dy, float* db, int N, int K, int PQ, float* workspace,
                       int64_t ws_bytes, bf_stream_t stream);
/* horizontally fused 1x1 stride-1 convolutions over the same x (Inception's
   1x1 / 3x3_reduce / 5x5_reduce, dispatcher fusion plan): one GEMM over the
   concatenated output channels, x read once.  Segment i (< 4): weights w[i]
   [kout[i]][C], bias b[i] (may be NULL), output y[i] (N, kout[i], H, W) and,
   if relu[i] != NULL, relu(y) into channels [relu_c0[i], relu_c0[i] + kout[i])
   of the relu_ctot[i]-channel tensor relu[i] (the fused relu_forward, possibly
   into a concat slice); y[i] may be NULL when relu[i] is not.  Host arrays of device pointers.  Same arithmetic per
   output as bf_conv2d_fwd_relu_slice (ops.py:281-297) */
int bf_conv1x1_fwd_group(const float* x, int N, int C, int H, int W, int nseg,
                         const float* const* w, const float* const* b, const int* kout,
                         float* const* y, float* const* relu, const int* relu_c0,
                         const int* relu_ctot, float* ws, int64_t ws_bytes, bf_stream_t stream);
/* the data gradients of such a group summed in one GEMM: dx = sum_i w[i]^T dy[i]
   over the K-concatenated dy[i] (N, kout[i], H, W) -- the Inception input
   gradient's three 1x1 parts, which the graph then aggregates with the pool
   branch's (ops.py:332-343 per part; the sum is reassociated: tolerance-level) */
int bf_conv1x1_dgrad_group(int N, int C, int H, int W, int nseg, const float* const* dy,
                           const float* const* w, const int* kout, float* dx, float* ws,
                           int64_t ws_bytes, bf_stream_t stream);
/* workspace bytes the conv/fc entry points want for this shape (0 = none) */
int64_t bf_gemm_workspace_bytes(int op, int N, int C, int H, int W, int K, int R, int S,
                                int P, int Q, int stride, int pad);

/* pooling (extension; Caffe ceil-mode geometry) -------------------------- */
int bf_maxpool_fwd(const float* x, float* y, float* mask, int N, int C, int H, int W,
                   int P, int Q, int kernel, int stride, int pad, bf_stream_t stream);
int bf_maxpool_bwd(const float* mask, const float* dy, float* dx, int N, int C, int H, int W,
                   int P, int Q, int kernel, int stride, int pad, bf_stream_t stream);
/* the same with relu_backward folded in: dx = (relu_x > 0 ? dx : 0), relu_x laid
   out as dx (the graph's following relu_backward and its dy tensor are elided) */
int bf_maxpool_bwd_relu(const float* mask, const float* dy, float* dx, const float* relu_x,
                        int N, int C, int H, int W, int P, int Q, int kernel, int stride, int pad,
                        bf_stream_t stream);
/* 3x3 max pooling staged through shared memory by bulk copies (pool_staged.cu).
   bf_maxpool_staged_ok: 1 when the shape is supported (backward 0: forward,
   1: the backward recomputing the argmax from x, 2: the backward reading the mask).  The
   forward writes the mask only when `mask` is non-null; the backward
   recomputes every window's argmax from x (bit-identical to the forward's) so
   the mask never has to be stored, and with relu_from_x != 0 applies the
   relu_backward of the operator that produced x = relu(a): dx = x > 0 ? dx : 0 */
int bf_maxpool_staged_ok(int N, int C, int H, int W, int P, int Q, int kernel, int stride,
                         int pad, int backward);
int bf_maxpool_fwd_staged(const float* x, float* y, float* mask, int N, int C, int H, int W,
                          int P, int Q, int kernel, int stride, int pad, bf_stream_t stream);
int bf_maxpool_bwd_x(const float* x, const float* dy, float* dx, int relu_from_x, int N, int C,
                     int H, int W, int P, int Q, int kernel, int stride, int pad,
                     bf_stream_t stream);
/* the same gather from the forward's mask (backward = 2 for bf_maxpool_staged_ok);
   bf_maxpool_bwd routes here where it fits */
int bf_maxpool_bwd_staged(const float* mask, const float* dy, float* dx, int N, int C, int H,
                          int W, int P, int Q, int kernel, int stride, int pad,
                          bf_stream_t stream);
/* signed argmax mask (backward = 3 for bf_maxpool_staged_ok: the forward and
   this backward both fit).  The forward writes y and, per window, the flat
   index of the first maximum when that maximum is > 0, -2 - index when it is
   <= 0, -1 when there is none ([N][C][P][Q] float32).  The backward gathers from
   it and dy only -- x is not read -- and with relu_from_sign != 0 applies the
   relu_backward of the operator that produced x = relu(a) from the sign
   (relu(a) > 0 <=> a > 0 at the argmax pixel; a pixel that is no window's
   argmax gets 0 either way): bit-identical to bf_maxpool_bwd_x */
int bf_maxpool_fwd_smask(const float* x, float* y, float* smask, int N, int C, int H, int W,
                         int P, int Q, int kernel, int stride, int pad, bf_stream_t stream);
int bf_maxpool_bwd_smask(const float* smask, const float* dy, float* dx, int relu_from_sign,
                         int N, int C, int H, int W, int P, int Q, int kernel, int stride, int pad,
                         bf_stream_t stream);
int bf_avgpool_fwd(const float* x, float* y, int N, int C, int H, int W, int P, int Q,
                   int kernel, int stride, int pad, bf_stream_t stream);
int bf_avgpool_bwd(const float* dy, float* dx, int N, int C, int H, int W, int P, int Q,
                   int kernel, int stride, int pad, bf_stream_t stream);

/* local response normalisation across channels (extension; Caffe) ------- */
/* scale may be NULL for size 5 (not stored: see bf_lrn_bwd_recompute) */
int bf_lrn_fwd(const float* x, float* y, float* scale, int N, int C, int H, int W, int size,
               float alpha, float beta, float k, bf_stream_t stream);
int bf_lrn_bwd(const float* x, const float* y, const float* scale, const float* dy, float* dx,
               int N, int C, int H, int W, int size, float alpha, float beta, float k,
               bf_stream_t stream);

int bf_lrn_bwd_relu(const float* x, const float* y, const float* scale, const float* dy,
                    float* dx, const float* relu_x, int N, int C, int H, int W, int size,
                    float alpha, float beta, float k, bf_stream_t stream);
/* graph-plan backward: scale and y recomputed from x with the forward's exact
   operation sequence (bit-identical to bf_lrn_bwd fed the forward's outputs),
   so the forward may run with scale == NULL; relu_x as bf_lrn_bwd_relu (NULL =
   none).  size 5 only. */
int bf_lrn_bwd_recompute(const float* x, const float* dy, float* dx, const float* relu_x, int N,
                         int C, int H, int W, int size, float alpha, float beta, float k,
                         bf_stream_t stream);

/* channel concat (extension); parts/channels are HOST arrays, k <= 32 ---- */
int bf_concat_fwd(const float* const* parts, const int* channels, int k, float* y,
                  int N, int H, int W, bf_stream_t stream);
int bf_concat_bwd(const float* dy, float* const* parts, const int* channels, int k,
                  int N, int H, int W, bf_stream_t stream);

/* NCCL over NVLink for the lowered parameter exchange (exchange.py) ----- */
int bf_nccl_unique_id(unsigned char out[128]);
int bf_nccl_init(void** comm, int nranks, int rank, const unsigned char id[128]);
int bf_nccl_destroy(void* comm);
int bf_nccl_reduce_scatter(void* comm, const float* send, float* recv, int64_t recv_count,
                           bf_stream_t stream);
int bf_nccl_all_gather(void* comm, const float* send, float* recv, int64_t send_count,
                       bf_stream_t stream);
int bf_nccl_all_reduce(void* comm, const float* send, float* recv, int64_t count,
                       bf_stream_t stream);

#ifdef __cplusplus
}
#endif

#endif /* PURINE_B200_H */
