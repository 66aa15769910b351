// gates.cu — the GRU "forward overhead" (FO; reading 10): the
// tape the GRU transposed Jacobian (eqn:gru_jcb) needs — h_{t-1},
// r, z, n and M = W_hn h_{t-1} + b_hn — recomputed from a forward that hides
// its gates (cuDNN).  Given every h_t, the recompute has no recurrence: all
// (t, b) rows at once, eqn:gru with torch's gate order (r, z, n):
//   r = sigma(W_ir x + b_ir + W_hr h_{t-1} + b_hr)
//   z = sigma(W_iz x + b_iz + W_hz h_{t-1} + b_hz)
//   M = W_hn h_{t-1} + b_hn,   n = tanh(W_in x + b_in + r M)
// One warp per row (grid-stride); the weights are staged once per CTA in
// shared memory, k-major (Ws[k][o], o < 3H), so a lane's output column reads
// are conflict-free and x / h_{t-1} are broadcast by shuffles.
#include "common.cuh"

namespace bppsa {
namespace {

constexpr int G_WARPS = 8;

__global__ void __launch_bounds__(32 * G_WARPS) gru_gates_kernel(int T, int B, int H, int I,
                                                                 const float* __restrict__ x,
                                                                 const float* __restrict__ h,
                                                                 const float* __restrict__ h_init,
                                                                 const float* __restrict__ Wih,
                                                                 const float* __restrict__ Whh,
                                                                 const float* __restrict__ bih,
                                                                 const float* __restrict__ bhh, float* __restrict__ hp_out,
                                                                 float* __restrict__ r_out, float* __restrict__ z_out,
                                                                 float* __restrict__ n_out, float* __restrict__ M_out) {
  extern __shared__ float sm[];
  const int O = 3 * H, K = I + H;
  float* Ws = sm;                                // [K][O]: k < I from W_ih3, else W_hh3
  float* gbuf = sm + K * O + (threadIdx.x >> 5) * 2 * O;   // per warp: gi [O], gh [O]
  for (int e = threadIdx.x; e < K * O; e += blockDim.x) {
    const int k = e / O, o = e % O;
    Ws[e] = k < I ? Wih[(long long)o * I + k] : Whh[(long long)o * H + (k - I)];
  }
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const long long rows = (long long)T * B;
  const long long warps = (long long)gridDim.x * G_WARPS;
  for (long long row = (long long)blockIdx.x * G_WARPS + (threadIdx.x >> 5); row < rows; row += warps) {
    const int t = (int)(row / B), b = (int)(row % B);
    // x (I <= 64: two per lane) and h_{t-1} (H <= 32: one per lane)
    float xv0 = 0.f, xv1 = 0.f, hv = 0.f;
    const float* xr = x + row * I;
    if (lane < I) xv0 = xr[lane];
    if (lane + 32 < I) xv1 = xr[lane + 32];
    const float* hprev = t > 0 ? h + (row - B) * H : (h_init ? h_init + (long long)b * H : nullptr);
    if (lane < H && hprev) hv = hprev[lane];
    float gi[3], gh[3];
#pragma unroll
    for (int j = 0; j < 3; ++j) {
      const int o = lane + 32 * j;
      gi[j] = (o < O) ? bih[o] : 0.f;
      gh[j] = (o < O) ? bhh[o] : 0.f;
    }
    for (int k = 0; k < I; ++k) {
      const float xk = __shfl_sync(0xffffffffu, k < 32 ? xv0 : xv1, k & 31);
#pragma unroll
      for (int j = 0; j < 3; ++j) {
        const int o = lane + 32 * j;
        if (o < O) gi[j] = fmaf(Ws[k * O + o], xk, gi[j]);
      }
    }
    for (int k = 0; k < H; ++k) {
      const float hk = __shfl_sync(0xffffffffu, hv, k);
#pragma unroll
      for (int j = 0; j < 3; ++j) {
        const int o = lane + 32 * j;
        if (o < O) gh[j] = fmaf(Ws[(I + k) * O + o], hk, gh[j]);
      }
    }
#pragma unroll
    for (int j = 0; j < 3; ++j) {
      const int o = lane + 32 * j;
      if (o < O) {
        gbuf[o] = gi[j];
        gbuf[O + o] = gh[j];
      }
    }
    __syncwarp();
    if (lane < H) {
      const int i = lane;
      const float r = 1.f / (1.f + expf(-(gbuf[i] + gbuf[O + i])));
      const float z = 1.f / (1.f + expf(-(gbuf[H + i] + gbuf[O + H + i])));
      const float M = gbuf[O + 2 * H + i];
      const float n = tanhf(gbuf[2 * H + i] + r * M);
      const long long off = row * H + i;
      hp_out[off] = hv;
      r_out[off] = r;
      z_out[off] = z;
      n_out[off] = n;
      M_out[off] = M;
    }
    __syncwarp();
  }
}

}  // namespace

cudaError_t launch_gru_gates(int T, int B, int H, int I, const float* x, const float* h, const float* h_init,
                             const float* Wih, const float* Whh, const float* bih, const float* bhh, float* hp,
                             float* r, float* z, float* n, float* M, int num_sms, cudaStream_t st) {
  const int O = 3 * H, K = I + H;
  const size_t smem = ((size_t)K * O + (size_t)G_WARPS * 2 * O) * sizeof(float);
  cudaError_t e = smem_attr_once(reinterpret_cast<const void*>(gru_gates_kernel), (int)smem);
  if (e != cudaSuccess) return e;
  const long long rows = (long long)T * B;
  const long long need = (rows + G_WARPS - 1) / G_WARPS;
  const int grid = (int)std::min<long long>(need, 4LL * num_sms);
  gru_gates_kernel<<<grid, 32 * G_WARPS, smem, st>>>(T, B, H, I, x, h, h_init, Wih, Whh, bih, bhh, hp, r, z, n, M);
  return cudaGetLastError();
}

}  // namespace bppsa
