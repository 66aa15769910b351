// Dev aid: 5D TMA load + store of the walk's box {32, 2, B, 1, G} (SW128) on a
// [T][B][64] fp32 array: copies one step of G blocks through shared memory.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 scripts/tma5d_probe.cu -o scripts/tma5d_probe.bin
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cuda.h>
__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__global__ void k(const __grid_constant__ CUtensorMap in, const __grid_constant__ CUtensorMap out, int c3, int c4, int mode) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(su32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(su32(&bar)), "r"(32768));
    if (mode == 0)
      asm volatile("cp.async.bulk.tensor.5d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5, %6}], [%7];\n"
                   ::"r"(su32(smem)), "l"(reinterpret_cast<uint64_t>(&in)), "r"(0), "r"(0), "r"(0), "r"(c3), "r"(c4), "r"(su32(&bar)) : "memory");
    else
      asm volatile("cp.async.bulk.tensor.5d.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5, %6}], [%7];\n"
                   ::"r"(su32(smem)), "l"(reinterpret_cast<uint64_t>(&in)), "r"(0), "r"(0), "r"(0), "r"(c3), "r"(c4), "r"(su32(&bar)) : "memory");
    asm volatile("{\n .reg .pred p;\nW:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n @!p bra W;\n}\n" ::"r"(su32(&bar)) : "memory");
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
    asm volatile("cp.async.bulk.tensor.5d.global.shared::cta.bulk_group [%0, {%1, %2, %3, %4, %5}], [%6];\n"
                 ::"l"(reinterpret_cast<uint64_t>(&out)), "r"(0), "r"(0), "r"(0), "r"(c3), "r"(c4), "r"(su32(smem)) : "memory");
    asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
    asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory");
  }
}
using Encode = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                            const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                            CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
int main() {
  const int T = 1000, B = 16, C = 64, G = 8;
  const long long A = (T - 1) / C;
  std::vector<float> h((size_t)T * B * 64), o(h.size(), -1.f);
  for (size_t i = 0; i < h.size(); ++i) h[i] = (float)i;
  float *dh, *dout;
  cudaMalloc(&dh, h.size() * 4); cudaMalloc(&dout, h.size() * 4);
  cudaMemcpy(dh, h.data(), h.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dout, o.data(), o.size() * 4, cudaMemcpyHostToDevice);
  void* fn; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  Encode enc = (Encode)fn;
  CUtensorMap mi, mo;
  const cuuint64_t dims[5] = {32, 2, (cuuint64_t)B, (cuuint64_t)C, (cuuint64_t)A};
  const cuuint64_t row = 256, strides[4] = {128, row, row * B, row * B * C};
  const cuuint32_t box[5] = {32u, 2u, (cuuint32_t)B, 1u, (cuuint32_t)G}, es[5] = {1, 1, 1, 1, 1};
  CUresult r1 = enc(&mi, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 5, dh, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                    CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  CUresult r2 = enc(&mo, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 5, dout, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                    CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encode %d %d\n", (int)r1, (int)r2);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 40 * 1024);
  for (int mode = 0; mode < 2; ++mode)
    for (int c4 : {3, -1}) {
      k<<<1, 32, 40 * 1024>>>(mi, mo, 5, c4, mode);
      cudaError_t e = cudaDeviceSynchronize();
      printf("mode %d c4 %d: %s\n", mode, c4, cudaGetErrorString(e));
      if (e != cudaSuccess) return 1;
    }
  cudaMemcpy(o.data(), dout, o.size() * 4, cudaMemcpyDeviceToHost);
  long bad = 0, copied = 0;
  for (size_t i = 0; i < o.size(); ++i) if (o[i] != -1.f) { ++copied; if (o[i] != h[i]) ++bad; }
  printf("copied %ld elements, %ld mismatched\n", copied, bad);
  return 0;
}
