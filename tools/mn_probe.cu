// Probe: TMA 3-D box load (128B swizzle) + one tcgen05.mma kind::tf32 with an
// MN-major A operand from shared memory, checked against a host GEMM.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_1412_6249_b200/csrc \
//        tools/mn_probe.cu -o tools/mn_probe.bin
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cmath>
#include <cstdio>
#include <vector>

#include "tc_ptx.cuh"

using namespace bf::tcu;

__device__ __forceinline__ uint64_t mn_desc(uint32_t saddr, int lbo, int sbo, int lt) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)lt << 61;
  return d;
}

// A: [32 k][128 m] as 4 boxes of [32 k][32 m]; B: K-major [N=32 rows][32 k] swizzled (host-packed)
__global__ void probe(const __grid_constant__ CUtensorMap amap, const float* bsw, float* araw,
                      float* out, int lbo, int sbo, int amajor, int lt) {
  __shared__ __align__(1024) uint8_t sm[16384 + 4096];
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t tslot;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 32;" ::"r"(
        smem_u32(&tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  for (int i = threadIdx.x; i < 1024; i += blockDim.x)
    reinterpret_cast<float*>(sm + 16384)[i] = bsw[i];
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tslot;
  if (threadIdx.x == 0) {
    mbar_arrive_expect_tx(&bar, 16384);
    for (int j = 0; j < 4; ++j)
      asm volatile(
          "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
          " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(smem_u32(sm + j * 4096)),
          "l"(reinterpret_cast<uint64_t>(&amap)), "r"(j * 32), "r"(0), "r"(0), "r"(smem_u32(&bar))
          : "memory");
    mbar_wait(&bar, 0);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) araw[i] = reinterpret_cast<float*>(sm)[i];
  if (threadIdx.x == 0) {
    const uint32_t idesc = tf32_idesc(32) | ((uint32_t)amajor << 15);
    const uint32_t a = smem_u32(sm), b = smem_u32(sm + 16384);
    for (int ks = 0; ks < 4; ++ks) {
      const uint64_t ad = mn_desc(a + ks * 1024, lbo, sbo, lt);
      const uint64_t bd = sw128_desc(b + ks * 32);
      if (ks == 0)
        asm volatile("tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, 0;" ::"r"(tmem),
                     "l"(ad), "l"(bd), "r"(idesc)
                     : "memory");
      else
        asm volatile("tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, 1;" ::"r"(tmem),
                     "l"(ad), "l"(bd), "r"(idesc)
                     : "memory");
    }
    tc_commit(&bar);
    mbar_wait(&bar, 1);
  }
  __syncthreads();
  tc_fence_after();
  {
    const int q = warp & 3;
    uint32_t v[16];
    for (int c0 = 0; c0 < 32; c0 += 16) {
      tmem_ld16(tmem + ((uint32_t)(q * 32) << 16) + c0, v);
      for (int j = 0; j < 16; ++j) out[(q * 32 + (threadIdx.x & 31)) * 32 + c0 + j] = __uint_as_float(v[j]);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 32;" ::"r"(tmem));
  }
}

int main() {
  // A logical [m = 128][k = 32]; global x[k][PQ = 128] (pixels contiguous)
  const int PQ = 128, K = 32, N = 32;
  std::vector<float> x(K * PQ), w(N * K), bsw(N * 32);
  for (int i = 0; i < K * PQ; ++i) x[i] = (float)((i * 37) % 17 - 8) * 0.125f;
  for (int i = 0; i < N * K; ++i) w[i] = (float)((i * 11) % 13 - 6) * 0.25f;
  // B K-major swizzled: row n (128 B = 32 k), chunk c (4 floats) at (c ^ (n & 7))
  for (int n = 0; n < N; ++n)
    for (int k = 0; k < K; ++k) {
      const int c = k / 4, e = k % 4;
      bsw[n * 32 + ((c ^ (n & 7)) * 4) + e] = w[n * K + k];
    }
  float *dx, *db, *draw, *dout;
  cudaMalloc(&dx, x.size() * 4);
  cudaMalloc(&db, bsw.size() * 4);
  cudaMalloc(&draw, 4096 * 4);
  cudaMalloc(&dout, 128 * 32 * 4);
  cudaMemcpy(dx, x.data(), x.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(db, bsw.data(), bsw.size() * 4, cudaMemcpyHostToDevice);
  void* p = nullptr;
  cudaDriverEntryPointQueryResult qr;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &qr);
  auto enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  CUtensorMap maps[2];
  for (int mi = 0; mi < 2; ++mi) {
    cuuint64_t dims[3] = {(cuuint64_t)PQ, (cuuint64_t)K, 1};
    cuuint64_t strides[2] = {(cuuint64_t)PQ * 4, (cuuint64_t)PQ * K * 4};
    cuuint32_t box[3] = {32, 32, 1}, es[3] = {1, 1, 1};
    CUresult r = enc(&maps[mi], CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, dx, dims, strides, box, es,
                     CU_TENSOR_MAP_INTERLEAVE_NONE,
                     mi ? CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B : CU_TENSOR_MAP_SWIZZLE_128B,
                     CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("encode %d rc %d\n", mi, (int)r);
  }
  std::vector<float> ref(128 * N);
  for (int m = 0; m < 128; ++m)
    for (int n = 0; n < N; ++n) {
      double s = 0;
      for (int k = 0; k < K; ++k) s += (double)x[k * PQ + m] * w[n * K + k];
      ref[m * N + n] = (float)s;
    }
  // {lbo, sbo, amajor, layout type, tma map}
  int cfg[][5] = {{4096, 512, 1, 1, 1}, {4096, 1024, 1, 1, 1}, {512, 4096, 1, 1, 1},
                  {4096, 1024, 0, 2, 0}};
  for (auto& c : cfg) {
    cudaMemset(dout, 0, 128 * 32 * 4);
    probe<<<1, 128>>>(maps[c[4]], db, draw, dout, c[0], c[1], c[2], c[3]);
    cudaError_t e = cudaDeviceSynchronize();
    std::vector<float> out(128 * 32), raw(4096);
    cudaMemcpy(out.data(), dout, out.size() * 4, cudaMemcpyDeviceToHost);
    cudaMemcpy(raw.data(), draw, raw.size() * 4, cudaMemcpyDeviceToHost);
    double err = 0;
    for (int i = 0; i < 128 * 32; ++i) err = fmax(err, fabs(out[i] - ref[i]));
    printf("lt %d amajor %d lbo %5d sbo %5d: %s maxerr %.3e  out[0..3] %.3f %.3f %.3f %.3f ref %.3f %.3f %.3f %.3f\n",
           c[3], c[2], c[0], c[1], cudaGetErrorString(e), err, out[0], out[1], out[2], out[3], ref[0], ref[1],
           ref[2], ref[3]);
    // smem layout check of box 0: row k, 128B; element (k, m) expected at chunk (m/4 ^ (k&7))
    int bad = 0;
    for (int k = 0; k < 32; ++k)
      for (int m = 0; m < 32; ++m) {
        const float got = raw[k * 32 + (((m / 4) ^ (k & 7)) * 4) + m % 4];
        if (got != x[k * PQ + m]) ++bad;
      }
    printf("   TMA box-0 layout mismatches vs [k][m] SW128: %d\n", bad);
  }
  return 0;
}
