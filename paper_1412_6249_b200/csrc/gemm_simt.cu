// SIMT fp32 implicit-GEMM engine (CUDA cores, exact fp32 FMA accumulation).
//
// Used for GEMM shapes the tcgen05 engine does not take (tiny or degenerate
// problems) and selectable via bf_set_gemm_engine(1) as an on-GPU cross-check
// of the tensor-core engine.  64x64x16 CTA tile, 256 threads, 4x4 outputs per
// thread, split-K over gridDim.z with an ordered (deterministic) reduction.
#include "gemm_common.cuh"
#include "gemm_engines.cuh"

namespace bf {
namespace {

constexpr int BM = 64, BN = 64, BK = 16, NT = 256;

template <class Ld>
__device__ __forceinline__ void load_tile(const Ld& ld, float (*dst)[BM + 4], int row0, int rows,
                                          int k0, int k1) {
#pragma unroll
  for (int i = 0; i < (BM * BK) / NT; ++i) {
    int e = threadIdx.x + i * NT;
    int r, kk;
    if (Ld::kMContig) {
      r = e % BM;
      kk = e / BM;
    } else {
      r = e / BK;
      kk = e % BK;
    }
    int gr = row0 + r, gk = k0 + kk;
    dst[kk][r] = (gr < rows && gk < k1) ? ld(gr, gk) : 0.f;
  }
}

template <class LA, class LB, class Epi>
__global__ void __launch_bounds__(NT) simt_gemm_kernel(LA la, LB lb, int M, int N, int K,
                                                       int k_per_split, Epi epi,
                                                       EpiPartial part, int splits) {
  __shared__ float As[BK][BM + 4];
  __shared__ float Bs[BK][BN + 4];
  int m0 = blockIdx.x * BM, n0 = blockIdx.y * BN;
  int kb = blockIdx.z * k_per_split;
  int ke = min(K, kb + k_per_split);
  int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
  float acc[4][4] = {};
  for (int k0 = kb; k0 < ke; k0 += BK) {
    load_tile(la, As, m0, M, k0, ke);
    load_tile(lb, Bs, n0, N, k0, ke);
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < BK; ++kk) {
      float4 a = *reinterpret_cast<const float4*>(&As[kk][ty * 4]);
      float4 b = *reinterpret_cast<const float4*>(&Bs[kk][tx * 4]);
      float av[4] = {a.x, a.y, a.z, a.w}, bv[4] = {b.x, b.y, b.z, b.w};
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(av[i], bv[j], acc[i][j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      int m = m0 + ty * 4 + i, n = n0 + tx * 4 + j;
      if (m < M && n < N) {
        if (splits > 1)
          part(blockIdx.z, m, n, acc[i][j]);
        else
          epi(m, n, acc[i][j]);
      }
    }
}

}  // namespace

template <class LA, class LB, class Epi>
int simt_gemm(const LA& la, const LB& lb, int M, int N, int K, const Epi& epi, float* ws,
              int64_t ws_bytes, cudaStream_t st, const char* what) {
  if (M <= 0 || N <= 0) return 0;
  int splits = choose_splits(M, N, K, BM, BN, 256, ws ? ws_bytes : 0);
  int kps = (K + splits - 1) / splits;
  kps = (kps + BK - 1) / BK * BK;
  splits = (K + kps - 1) / kps;
  if (splits < 1) splits = 1;
  dim3 grid((M + BM - 1) / BM, (N + BN - 1) / BN, splits);
  EpiPartial part{ws, M, N};
  simt_gemm_kernel<LA, LB, Epi><<<grid, NT, 0, st>>>(la, lb, M, N, K, kps, epi, part, splits);
  if (int rc = check_launch(what)) return rc;
  if (splits > 1) {
    splitk_reduce<Epi>(ws, splits, M, N, epi, st);
    return check_launch(what);
  }
  return 0;
}

// explicit instantiations used by gemm_api.cu
#define BF_SIMT_INST(LA, LB, EPI) \
  template int simt_gemm<LA, LB, EPI>(const LA&, const LB&, int, int, int, const EPI&, float*, \
                                      int64_t, cudaStream_t, const char*);
BF_SIMT_INST(LdFwdX, LdRowK, EpiNCHW)
BF_SIMT_INST(LdDgradDY, LdDgradW, EpiNCHW)
BF_SIMT_INST(LdWgradX, LdWgradDY, EpiT)
BF_SIMT_INST(LdColK, LdRowK, EpiT)
BF_SIMT_INST(LdRowK, LdRowK, EpiT)
BF_SIMT_INST(LdColK, LdColK, EpiT)

}  // namespace bf
