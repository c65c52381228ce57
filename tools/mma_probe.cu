// Microbenchmark: raw tcgen05.mma kind::tf32 issue rate on one SM-resident CTA
// per SM, A from TMEM ("ts") or shared memory ("ss"), for N = 32..256, with and
// without the per-k-block mbarrier round trip the GEMM engines use.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../paper_1412_6249_b200/csrc \
//        tools/mma_probe.cu -o /tmp/mma_probe && /tmp/mma_probe
//
// Prints cycles per MMA instruction and the implied TF32 TFLOP/s over 148 SMs.
#include <cstdio>
#include <cstdint>

#include "tc_ptx.cuh"

using namespace bf::tcu;

__device__ __forceinline__ void mma_ss(uint32_t d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                       uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(acc)
      : "memory");
}

// mode 0: ts back-to-back; 1: ss back-to-back; 2: ts with a commit + wait every `per` MMAs;
// 3: ts round-robin over `per` independent accumulators (columns n*j)
__global__ void probe(int n, int iters, int mode, int per, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint32_t tslot;
  __shared__ __align__(8) uint64_t bar;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
        smem_u32(&tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  for (int i = threadIdx.x; i < 64 * 1024 / 4; i += blockDim.x)
    reinterpret_cast<float*>(smem)[i] = 1.0f / (1 + (i & 7));
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tslot;
  unsigned long long t0 = 0, t1 = 0;
  if (mode >= 8) {  // `per` issuing warps (lane 0 each), each into its own accumulator
    __shared__ __align__(8) uint64_t bars[4];
    if (threadIdx.x == 0) {
      for (int b = 0; b < 4; ++b) mbar_init(&bars[b], 1);
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (warp < per && (threadIdx.x & 31) == 0) {
      const uint32_t idesc = tf32_idesc(n);
      const uint32_t bsm = smem_u32(smem);
      uint64_t bdv[4];
      for (int k = 0; k < 4; ++k) bdv[k] = sw128_desc(bsm + k * 32);
      const uint32_t dcol = tmem + (uint32_t)(warp * (256 / per)), acol = tmem + 256 + warp * 32;
      mma_ts(dcol, acol, bdv[0], idesc, 0u);
      const unsigned long long s0 = clock64();
      for (int i = 0; i < iters / per; i += 8) {
#pragma unroll
        for (int u = 0; u < 8; ++u)
          asm volatile("tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, 1;" ::"r"(dcol),
                       "r"(acol + (u & 3) * 8), "l"(bdv[u & 3]), "r"(idesc)
                       : "memory");
      }
      tc_commit(&bars[warp]);
      mbar_wait(&bars[warp], 0);
      const unsigned long long s1 = clock64();
      if (warp == 0) out[blockIdx.x] = s1 - s0;
    }
  } else if (threadIdx.x == 0) {
    const uint32_t idesc = tf32_idesc(n);
    const uint32_t bsm = smem_u32(smem);
    const uint32_t asm_ = bsm + 32768;
    uint32_t phase = 0;
    if (mode >= 6) {  // GEMM-like k-blocks: 12 MMAs + `per` commits (6: commit, 7: +wait-free mbar check)
      __shared__ __align__(8) uint64_t dummy[2];
      if (true) {
        mbar_init(&dummy[0], 1);
        mbar_init(&dummy[1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
      }
      const uint64_t db = sw128_desc(bsm), ds = db + (uint64_t)((n * 128) >> 4);
      const uint32_t ab = tmem + 256;
      mma_ts_flag<0>(tmem, ab, db, idesc);
      t0 = clock64();
      for (int i = 0; i < iters; i += 12) {
#pragma unroll
        for (int ks = 0; ks < 4; ++ks) {
          const uint64_t k2 = (uint64_t)((ks * 32) >> 4);
          mma_ts_flag<1>(tmem, ab + 32 + ks * 8, db + k2, idesc);
          mma_ts_flag<1>(tmem, ab + ks * 8, ds + k2, idesc);
          mma_ts_flag<1>(tmem, ab + ks * 8, db + k2, idesc);
        }
        for (int c = 0; c < per; ++c) tc_commit(&dummy[c & 1]);
      }
      tc_commit(&bar);
      mbar_wait(&bar, 0);
      t1 = clock64();
      out[blockIdx.x] = t1 - t0;
    } else if (mode >= 4) {  // straight-line issue: precomputed descriptors, constant accumulate flag
      uint64_t bdv[4];
      for (int k = 0; k < 4; ++k) bdv[k] = sw128_desc(bsm + k * 32);
      const uint32_t dcol = tmem, acol = tmem + 256;
      mma_ts(dcol, acol, bdv[0], idesc, 0u);
      t0 = clock64();
      for (int i = 0; i < iters; i += 8) {
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const uint32_t d = mode == 5 ? dcol + (uint32_t)((u & 1) * n) : dcol;
          asm volatile("tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, 1;" ::"r"(d),
                       "r"(acol + (u & 3) * 8), "l"(bdv[u & 3]), "r"(idesc)
                       : "memory");
        }
      }
      tc_commit(&bar);
      mbar_wait(&bar, 0);
      t1 = clock64();
      out[blockIdx.x] = t1 - t0;
    } else {
    t0 = clock64();
    for (int i = 0; i < iters; ++i) {
      const int ks = i & 3;
      const uint64_t bd = sw128_desc(bsm + ks * 32);
      if (mode == 1)
        mma_ss(tmem, sw128_desc(asm_ + ks * 32), bd, idesc, i > 0);
      else if (mode == 3)
        mma_ts(tmem + (uint32_t)((i % per) * n), tmem + 448 + ks * 8, bd, idesc, i >= per);
      else
        mma_ts(tmem, tmem + 256 + ks * 8, bd, idesc, i > 0);
      if (mode == 2 && (i % per) == per - 1) {
        tc_commit(&bar);
        mbar_wait(&bar, phase);
        phase ^= 1;
      }
    }
    tc_commit(&bar);
    mbar_wait(&bar, phase);
    t1 = clock64();
    out[blockIdx.x] = t1 - t0;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
  }
}

int main() {
  unsigned long long* d;
  cudaMalloc(&d, 148 * sizeof(unsigned long long));
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  int clk = 0;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  const int iters = 8192;
  struct Cfg { const char* name; int mode, per; };
  const Cfg cfgs[] = {{"ts", 0, 1}, {"ss", 1, 1}, {"ts+sync/12", 2, 12}, {"ts x2 acc", 3, 2},
                      {"ts unrolled", 4, 1}, {"ts unr x2acc", 5, 2}, {"kblk 0 commit", 6, 0},
                      {"kblk 1 commit", 6, 1}, {"kblk 2 commit", 6, 2},
                      {"2 issuers", 8, 2}, {"4 issuers", 8, 4}};
  for (const Cfg& c : cfgs) {
    for (int n : {32, 64, 128, 192, 256}) {
      if ((c.mode == 3 || c.mode == 5 || c.mode == 8) && c.per * n > 256) continue;
      probe<<<148, 128, 100 * 1024>>>(n, iters, c.mode, c.per, d);
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) {
        printf("error %s\n", cudaGetErrorString(e));
        return 1;
      }
      unsigned long long h[148];
      cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
      double mx = 0;
      for (int i = 0; i < 148; ++i) mx = h[i] > mx ? h[i] : mx;
      const double cyc = mx / iters;
      const double flops = 2.0 * 128 * n * 8;
      printf("%-11s N=%3d  %7.1f cycles/MMA  %7.1f TFLOP/s tf32 (at %d MHz)\n", c.name, n, cyc,
             flops / cyc * 148 * clk * 1e3 / 1e12, clk / 1000);
    }
  }
  return 0;
}
