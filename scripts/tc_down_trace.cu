// Dev aid: per-step phase timestamps (clock64) of the 3xFP16 level-0 walk on
// CTA 0 (slot 0/1, warps 0 and 5).  Build + run on a B200:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o scripts/tc_down_trace.bin scripts/tc_down_trace.cu && scripts/tc_down_trace.bin
#define BPPSA_STEP_TRACE 1
#include <algorithm>
#include <cstdio>
#include <vector>
#include "../paper_1907_10134_b200/csrc/tc_leaf.cu"

int main() {
  const int T = 1 << 18, B = 16, H = 64, C = 512;
  std::vector<float> h((size_t)T * B * H), W(H * H), seed(B * H);
  unsigned s = 1;
  auto rnd = [&] { s = s * 1664525u + 1013904223u; return (s >> 8) / 16777216.f; };
  for (auto& v : h) v = rnd() * 1.6f - 0.8f;
  for (auto& v : W) v = (rnd() * 2 - 1) / 8.f;
  for (auto& v : seed) v = rnd() - 0.5f;
  const long long nblk = (T + 1 + C - 1) / C;
  float *dh, *dW, *dcarry, *dg, *dseed;
  cudaMalloc(&dh, h.size() * 4); cudaMalloc(&dW, W.size() * 4); cudaMalloc(&dseed, seed.size() * 4);
  cudaMalloc(&dcarry, (size_t)B * nblk * H * 4); cudaMalloc(&dg, h.size() * 4);
  cudaMemcpy(dh, h.data(), h.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dW, W.data(), W.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dseed, seed.data(), seed.size() * 4, cudaMemcpyHostToDevice);
  cudaMemset(dcarry, 0, (size_t)B * nblk * H * 4);
  bppsa::LeafArgs a{};
  a.seg = bppsa::Seg{T, B, H, 1};
  a.kind = BPPSA_JAC_RNN_TANH;
  a.h = dh; a.W = dW; a.seed = dseed;
  for (int rep = 0; rep < 2; ++rep) bppsa::launch_tc_leaf_down(a, C, dcarry, nblk, dg, nullptr, 148, 0);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  bppsa::launch_tc_leaf_down(a, C, dcarry, nblk, dg, nullptr, 148, 0);
  cudaEventRecord(e1);
  cudaError_t err = cudaDeviceSynchronize();
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  printf("status %s  time %.3f ms (T=%d, C=%d)\n", cudaGetErrorString(err), ms, T, C);
  static long long tr[2][2][8][4096];
  cudaMemcpyFromSymbol(tr, bppsa::g_step_trace, sizeof(tr));
  const char* names[] = {"top", "D+h ready", "D read", "grad stored", "A stored", "after bar3", "issued+max"};
  for (int g = 0; g < 2; ++g)
    for (int w = 0; w < 2; ++w) {
      printf("slot %d warp %s:", g, w ? "5" : "0");
      for (int p = 1; p <= 6; ++p) {
        std::vector<long long> d;
        for (int st = 50; st < 400; ++st) d.push_back(tr[g][w][p][st] - tr[g][w][p - 1][st]);
        std::sort(d.begin(), d.end());
        printf("  %s->%s %lld", names[p - 1], names[p], d[d.size() / 2]);
      }
      std::vector<long long> d;
      for (int st = 50; st < 400; ++st) d.push_back(tr[g][w][0][st + 1] - tr[g][w][0][st]);
      std::sort(d.begin(), d.end());
      printf("  | step %lld\n", d[d.size() / 2]);
    }
  return 0;
}
