// Dev aid: issue throughput of the fp16 split instructions on sm_100a
// (F2FP.F16.F32.PACK_AB, HADD2.F32 unpack, FMUL2/FADD2) vs FFMA / integer ops,
// alone and interleaved (do they share a pipe?).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o scripts/op_rate.bin scripts/op_rate.cu
#include <cstdio>
#include <cuda_fp16.h>
__device__ __forceinline__ float f2fp(float a, float b) {
  unsigned r;
  asm volatile("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(a), "f"(b));
  return __uint_as_float(r);
}
__device__ __forceinline__ float ffma_(float a, float b) {
  float r;
  asm volatile("fma.rn.f32 %0, %1, %2, 0f3F000000;" : "=f"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ float iop(float a) {
  unsigned r;
  asm volatile("{.reg .u32 t; add.u32 t, %1, 4096; and.b32 %0, t, 0xFFFFE000;}" : "=r"(r) : "r"(__float_as_uint(a)));
  return __uint_as_float(r);
}
__device__ __forceinline__ float h2f(float a) {
  float r;
  asm volatile("{.reg .b16 lo, hi; mov.b32 {lo, hi}, %1; cvt.f32.f16 %0, lo;}" : "=f"(r) : "r"(__float_as_uint(a)));
  return r;
}
template <int OP>
__global__ void k(float* out, int iters) {
  float a[8], b[8], c[8];
  for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 0.001f + i, b[i] = 1.0001f + i * 1e-5f, c[i] = a[i] * 0.5f;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (OP == 0) a[i] = ffma_(a[i], b[i]);
      if (OP == 1) a[i] = f2fp(a[i], b[i]);
      if (OP == 2) a[i] = h2f(a[i]);
      if (OP == 3) a[i] = iop(a[i]);
      if (OP == 4) { a[i] = f2fp(a[i], b[i]); c[i] = ffma_(c[i], b[i]); }
      if (OP == 5) { a[i] = f2fp(a[i], b[i]); c[i] = iop(c[i]); }
      if (OP == 6) { a[i] = h2f(a[i]); c[i] = ffma_(c[i], b[i]); }
      if (OP == 7) { a[i] = ffma_(a[i], b[i]); c[i] = iop(c[i]); }
    }
  }
  long long t1 = clock64();
  float s = 0;
  for (int i = 0; i < 8; ++i) s += a[i] + b[i] + c[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = (float)(t1 - t0);
}
template <int OP>
void run(const char* name, float* d) {
  const int iters = 4096;
  k<OP><<<148, 1024>>>(d, iters);
  cudaDeviceSynchronize();
  float cyc;
  cudaMemcpy(&cyc, d, 4, cudaMemcpyDeviceToHost);
  printf("%-16s %.3f cycles per iteration-slot per SM (8 x 32 warps per iteration)\n", name, cyc / (iters * 8.0 * 32));
}
int main() {
  float* d;
  cudaMalloc(&d, 148 * 1024 * 4);
  run<0>("FFMA", d);
  run<1>("F2FP", d);
  run<2>("HADD2.F32", d);
  run<3>("IADD+LOP", d);
  run<4>("F2FP+FFMA", d);
  run<5>("F2FP+IADD+LOP", d);
  run<6>("HADD2+FFMA", d);
  run<7>("FFMA+IADD+LOP", d);
  return 0;
}
