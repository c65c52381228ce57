// GEMM engine entry points (templated on loaders / epilogue).
#pragma once

#include "gemm_common.cuh"

namespace bf {

// SIMT fp32 engine (gemm_simt.cu)
template <class LA, class LB, class Epi>
int simt_gemm(const LA& la, const LB& lb, int M, int N, int K, const Epi& epi, float* ws,
              int64_t ws_bytes, cudaStream_t st, const char* what);

// tcgen05 3xTF32 engine (gemm_tc.cu); returns -1 when the shape is not taken
template <class LA, class LB, class Epi>
int tc_gemm(const LA& la, const LB& lb, int M, int N, int K, const Epi& epi, float* ws,
            int64_t ws_bytes, cudaStream_t st, const char* what);

// tcgen05 engine v2 (gemm_tc2.cu): A in TMEM, pre-packed B via bulk TMA
int tc2_conv_fwd(const LdFwdX& la, const LdRowK& lb, int M, int N, int K, const EpiNCHW& epi,
                 float* ws, int64_t ws_bytes, cudaStream_t st, const char* what);
int tc2_conv_dgrad(const LdDgradDY& la, const LdDgradW& lb, int M, int N, int K,
                   const EpiNCHW& epi, float* ws, int64_t ws_bytes, cudaStream_t st,
                   const char* what);
// db != NULL: the bias gradient is fused into the dY pack when the fast path is
// taken (*db_done = true); otherwise the caller computes it
int tc2_conv_wgrad(const LdWgradX& la, const LdWgradDY& lb, int M, int N, int K,
                   const EpiT& epi, float* ws, int64_t ws_bytes, cudaStream_t st,
                   const char* what, float* db = nullptr, bool* db_done = nullptr);

// tcgen05 engine v3 (gemm_tc3.cu): halo-staged stride-1 R x S convolutions
int tc3_conv_fwd(const ConvShape& g, const float* x, const float* w, const EpiNCHW& epi,
                 float* ws, int64_t ws_bytes, cudaStream_t st, const char* what);
int tc3_conv_dgrad(const ConvShape& g, const float* dy, const float* w, const EpiNCHW& epi,
                   float* ws, int64_t ws_bytes, cudaStream_t st, const char* what);

// tcgen05 engine v4 (gemm_tc4.cu): TMA-fed 1x1 convolutions (MN-major activation operand)
int tc4_conv_fwd(const ConvShape& g, const float* x, const float* w, const EpiNCHW& epi,
                 float* ws, int64_t ws_bytes, cudaStream_t st, const char* what);
int tc4_conv_dgrad(const ConvShape& g, const float* dy, const float* w, const EpiNCHW& epi,
                   float* ws, int64_t ws_bytes, cudaStream_t st, const char* what);
// grouped 1x1 data gradients of convolutions over the same x: one GEMM over the
// K-concatenated dy segments (each padded to 32 channels), i.e. their SUM
int tc4_conv_dgrad_group(int N, int C, int HW, int nseg, const float* const* dy,
                         const float* const* w, const int* kout, const EpiNCHW& epi, float* ws,
                         int64_t ws_bytes, cudaStream_t st, const char* what);
// horizontally fused 1x1 forward convolutions over the same x (segmented epilogue)
int tc4_conv_fwd_group(const float* x, int N, int C, int HW, int nseg, const float* const* w,
                       const int* kout, const EpiNCHWSeg& epi, float* ws, int64_t ws_bytes,
                       cudaStream_t st, const char* what);

// strided convolutions (C*stride^2 <= 64 channels, kernel wider than the
// stride) as stride-1 convolutions over a space-to-depth view (conv_s2d.cu)
bool s2d_enabled();  // PURINE_B200_S2D=1 (opt-in)
int s2d_conv_fwd(const ConvShape& g, const float* x, const float* w, const EpiNCHW& epi,
                 float* ws, int64_t ws_bytes, cudaStream_t st, const char* what);
int s2d_conv_wgrad(const ConvShape& g, const float* x, const float* dy, float* dw, float* db,
                   bool* db_done, float* ws, int64_t ws_bytes, cudaStream_t st,
                   const char* what);

// transposed weight gradient for few-input-channel convolutions (conv1):
// D[kout][(c,r,s)] with dY by TMA and the im2col from contiguous windows
// (gemm_wgrad_t.cu); -1 when not taken
int wgrad_t_conv(const ConvShape& g, const float* x, const float* dy, float* dw, float* db,
                 bool* db_done, float* ws, int64_t ws_bytes, cudaStream_t st, const char* what);

// forward of a few-input-channel convolution (conv1) from contiguous input-row
// windows, weights resident in shared memory (gemm_fwd_win.cu); -1 when not taken
int fwd_win_conv(const ConvShape& g, const float* x, const float* w, const EpiNCHW& epi,
                 float* ws, int64_t ws_bytes, cudaStream_t st, const char* what);

extern int g_gemm_engine;  // 0 auto, 1 simt, 2 tcgen05 v1 only, 3 auto + halo engine v3 (opt-in),
                           // 4 auto without v4, 5 auto without the TMA-fed 1x1 weight gradient,
                           // 6 auto with register-prefetched (not cp.async-staged) gathers,
                           // 7 auto + TMA-streamed raw dY for conv1-type weight gradients
// the TMA-fed 1x1 weight gradient (engine v2 mode kTma1x1) is taken unless engine 5
inline bool tc2_tma_wgrad_enabled() { return g_gemm_engine != 5; }
// engine v2's gathers staged AD k-blocks ahead through cp.async unless engine 6
inline bool tc2_async_gather_enabled() { return g_gemm_engine != 6; }
// weight gradients whose output rows are 16-byte multiples stream the raw dY
// by TMA (mode kWgradTma: no dY pack; the epilogue warps split the B tile).
// Default on (PURINE_B200_WGRAD_TMA=0 disables); off with engines 4-6.
// (Round 1's form, with the issue-bound producers splitting the B tile, was
// neutral in the step and 5% slower alone.)
bool tc2_wgrad_tma_enabled();
// weight-gradient units split-major (PURINE_B200_SPLIT_OUTER, default 1)
bool tc2_split_outer();
// widest tile given a separate small-term accumulator (PURINE_B200_SACC=0: none;
// PURINE_B200_SACC_MAX_BN, default 128)
int tc2_sacc_max_bn();

}  // namespace bf
