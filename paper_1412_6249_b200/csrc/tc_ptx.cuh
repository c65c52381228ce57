// tcgen05 / TMA / mbarrier PTX helpers shared by the tcgen05 engines v2 (gemm_tc2.cu)
// and v3 (gemm_tc3.cu).  sm_100a only.
#pragma once

#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstdint>

namespace bf {
namespace tcu {

constexpr int BM = 128;  // accumulator rows = TMEM lanes

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.expect_tx.relaxed.cta.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
// arrive (count 1) and add the expected transaction bytes in one step
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@!P1 bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes,
                                         uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
          "r"(dst),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
// TMA tiled load of a 3-D box into shared memory, completing on ``bar``
__device__ __forceinline__ void tma_load_3d(uint32_t dst, const CUtensorMap* map, int c0, int c1,
                                            int c2, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
      : "memory");
}

// TMA tiled load of a 4-D box into shared memory, completing on ``bar``
__device__ __forceinline__ void tma_load_4d(uint32_t dst, const CUtensorMap* map, int c0, int c1,
                                            int c2, int c3, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4, %5}], [%6];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(c3),
      "r"(smem_u32(bar))
      : "memory");
}

// cuTensorMapEncodeTiled through the runtime's driver entry point (no libcuda link)
static inline PFN_cuTensorMapEncodeTiled_v12000 tma_encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

// [imgs][rows][PQ] fp32 NCHW activation viewed 3-D; box {32 pixels, box_rows, 1}
static inline bool make_nchw_map(CUtensorMap* map, const float* p, int PQ, int rows, int imgs,
                                 int box_rows, CUtensorMapSwizzle swz) {
  auto fn = tma_encode_fn();
  if (!fn) return false;
  cuuint64_t dims[3] = {(cuuint64_t)PQ, (cuuint64_t)rows, (cuuint64_t)imgs};
  cuuint64_t strides[2] = {(cuuint64_t)PQ * 4, (cuuint64_t)PQ * rows * 4};
  cuuint32_t box[3] = {32, (cuuint32_t)box_rows, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  return fn(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float*>(p), dims, strides, box,
            estr, CU_TENSOR_MAP_INTERLEAVE_NONE, swz, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// one lane of a converged warp (the lowest active); the same lane every call
__device__ __forceinline__ bool elect_one() {
  uint32_t pred = 0;
  asm volatile(
      "{\n\t.reg .pred P;\n\telect.sync _|P, 0xffffffff;\n\tselp.u32 %0, 1, 0, P;\n\t}"
      : "=r"(pred));
  return pred != 0;
}
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_u32(bar))
               : "memory");
}
// D[tmem] (+)= A[tmem] * B[smem desc]
__device__ __forceinline__ void mma_ts(uint32_t d, uint32_t a, uint64_t bdesc, uint32_t idesc,
                                       uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d),
      "r"(a), "l"(bdesc), "r"(idesc), "r"(acc)
      : "memory");
}
// same with a compile-time accumulate flag (no per-instruction predicate setup)
template <int ACC>
__device__ __forceinline__ void mma_ts_flag(uint32_t d, uint32_t a, uint64_t bdesc,
                                            uint32_t idesc) {
  asm volatile("tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, %4;" ::"r"(d), "r"(a),
               "l"(bdesc), "r"(idesc), "n"(ACC)
               : "memory");
}
__device__ __forceinline__ void tmem_st16(uint32_t taddr, const float (&v)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(taddr),
      "f"(v[0]), "f"(v[1]), "f"(v[2]), "f"(v[3]), "f"(v[4]), "f"(v[5]), "f"(v[6]), "f"(v[7]),
      "f"(v[8]), "f"(v[9]), "f"(v[10]), "f"(v[11]), "f"(v[12]), "f"(v[13]), "f"(v[14]),
      "f"(v[15])
      : "memory");
}
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&v)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
        "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]),
        "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void named_sync(int id, int count) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(count) : "memory");
}
__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)1 << 16;
  d |= (uint64_t)(1024 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}
__device__ __forceinline__ uint32_t tf32_idesc(int bn) {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(bn >> 3) << 17) |
         ((uint32_t)(BM >> 4) << 24);
}
// round to the nearest TF32 value (ties away from zero) in two integer ops:
// add half a TF32 ulp to the magnitude bits, clear the 13 dropped bits
__device__ __forceinline__ float to_tf32_rna(float x) {
  return __uint_as_float((__float_as_uint(x) + 0x1000u) & 0xFFFFE000u);
}
// Small part of the implicit 3xTF32 split of a raw fp32 operand.  The tensor
// core reads a kind::tf32 operand's fp32 bits and ignores the 13 low mantissa
// bits, so big = x as is stands for trunc(x), and s = x - trunc(x) is exact in
// fp32.  The MMA then truncates s in turn; that error always has the sign of
// x (|A| shrinks by up to 2^-20 |x|), a coherent bias that adds up over long
// reductions and network depth.  TF32_SMALL_RNA (default) adds half a TF32
// ulp to s's magnitude bits so the MMA's truncation rounds s to nearest
// instead: unbiased, error <= 2^-21 |x|, one integer add per element.
#ifndef TF32_SMALL_RNA
#define TF32_SMALL_RNA 1
#endif
__device__ __forceinline__ float tf32_small(float x) {
  const float s = x - __uint_as_float(__float_as_uint(x) & 0xFFFFE000u);
#if TF32_SMALL_RNA
  return __uint_as_float(__float_as_uint(s) + 0x1000u);
#else
  return s;
#endif
}
__device__ __forceinline__ float4 tf32_small4(float4 v) {
  return make_float4(tf32_small(v.x), tf32_small(v.y), tf32_small(v.z), tf32_small(v.w));
}
__device__ __forceinline__ uint32_t sw_off(int r, int c) {
  return (uint32_t)(r * 128 + (((c ^ r) & 7) << 4));
}

// ---- B pre-pack: [n_tile][k_block][big BN x 128B | small BN x 128B], swizzled ----

// one thread per 16-byte chunk (row r of the tile, 4 consecutive k): grid
// (k-blocks, n-tiles, BN/32) so even a small weight tensor spreads over
// enough CTAs to be latency- rather than CTA-count-bound
template <class LB>
__global__ void pack_b_kernel(LB lb, int N, int K, int BN, int nkb, uint8_t* __restrict__ out) {
  const int tile = blockIdx.y, kb = blockIdx.x;
  uint8_t* base = out + ((size_t)tile * nkb + kb) * 2 * BN * 128;
  const int i = blockIdx.z * blockDim.x + threadIdx.x;
  if (i >= BN * 8) return;
  const int r = i >> 3, c = i & 7;
  const int n = tile * BN + r;
  float v[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const int k = kb * 32 + c * 4 + j;
    v[j] = (n < N && k < K) ? lb(n, k) : 0.f;
  }
  float4 bg, sm;
  bg.x = to_tf32_rna(v[0]); sm.x = to_tf32_rna(v[0] - bg.x);
  bg.y = to_tf32_rna(v[1]); sm.y = to_tf32_rna(v[1] - bg.y);
  bg.z = to_tf32_rna(v[2]); sm.z = to_tf32_rna(v[2] - bg.z);
  bg.w = to_tf32_rna(v[3]); sm.w = to_tf32_rna(v[3] - bg.w);
  const uint32_t off = sw_off(r, c);
  *reinterpret_cast<float4*>(base + off) = bg;
  *reinterpret_cast<float4*>(base + BN * 128 + off) = sm;
}

template <class LB>
inline void launch_pack_b(const LB& lb, int N, int K, int BN, int nkb, int ntiles, uint8_t* out,
                          cudaStream_t st) {
  pack_b_kernel<LB><<<dim3(nkb, ntiles, (BN * 8 + 255) / 256), 256, 0, st>>>(lb, N, K, BN, nkb,
                                                                            out);
}

// db[ko] = sum over k-blocks of the per-block partials (weight-gradient engines), in a fixed order
// (strided per thread, then a shared-memory tree): deterministic
static __global__ void bias_blocks_finish_kernel(const float* __restrict__ part, int nkb,
                                          float* __restrict__ db) {
  __shared__ float red[256];
  const float* row = part + (size_t)blockIdx.x * nkb;
  // four independent strided chains per thread (loads in flight), combined in a
  // fixed order, then a fixed shared-memory tree
  float acc[4] = {0.f, 0.f, 0.f, 0.f};
  for (int kb = threadIdx.x; kb < nkb; kb += 4 * 256) {
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int k = kb + u * 256;
      if (k < nkb) acc[u] = __fadd_rn(acc[u], __ldg(row + k));
    }
  }
  red[threadIdx.x] = __fadd_rn(__fadd_rn(acc[0], acc[1]), __fadd_rn(acc[2], acc[3]));
  __syncthreads();
  for (int s = 128; s > 0; s >>= 1) {
    if (threadIdx.x < s) red[threadIdx.x] = __fadd_rn(red[threadIdx.x], red[threadIdx.x + s]);
    __syncthreads();
  }
  if (threadIdx.x == 0) db[blockIdx.x] = red[0];
}

}  // namespace tcu
}  // namespace bf
