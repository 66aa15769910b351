// Dev aid: per-step phase timestamps (clock64) of the 16-warp tcgen05 level-0
// up-sweep on CTA 0.  Build + run on a B200:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o /tmp/tr scripts/tc_up_trace.cu && /tmp/tr
#define BPPSA_STEP_TRACE 1
#include <cstdio>
#include <vector>
#include <algorithm>
#include "../paper_1907_10134_b200/csrc/tc_leaf.cu"

int main(int argc, char** argv) {
  const int prec = argc > 1 ? atoi(argv[1]) : 0;   // 0 = 3xFP16, 1 = 3xTF32
  const int T = 1 << 18, B = 16, H = 64, C = 256;
  std::vector<float> h((size_t)T * B * H), W(H * H);
  unsigned s = 1;
  auto rnd = [&] { s = s * 1664525u + 1013904223u; return (s >> 8) / 16777216.f; };
  for (auto& v : h) v = rnd() * 1.6f - 0.8f;
  for (auto& v : W) v = (rnd() * 2 - 1) / 8.f;
  float *dh, *dW, *dagg;
  cudaMalloc(&dh, h.size() * 4); cudaMalloc(&dW, W.size() * 4);
  const long long nblk = T / C;
  cudaMalloc(&dagg, (size_t)B * nblk * H * H * 4);
  cudaMemcpy(dh, h.data(), h.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dW, W.data(), W.size() * 4, cudaMemcpyHostToDevice);
  bppsa::LeafArgs a{};
  a.seg = bppsa::Seg{T, B, H, 0};
  a.kind = BPPSA_JAC_RNN_TANH;
  a.h = dh; a.W = dW;
  for (int rep = 0; rep < 2; ++rep) bppsa::launch_tc_leaf_up(a, C, dagg, nblk, 0, 148, 0, prec);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  bppsa::launch_tc_leaf_up(a, C, dagg, nblk, 0, 148, 0, prec);
  cudaEventRecord(e1);
  cudaError_t err = cudaDeviceSynchronize();
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  printf("prec %d status %s  time %.3f ms (T=%d)\n", prec, cudaGetErrorString(err), ms, T);
  static long long tr[2][2][8][4096];
  cudaMemcpyFromSymbol(tr, bppsa::g_step_trace, sizeof(tr));
  const char* names[] = {"start", "A stored", "after bar", "issued", "D ready", "D loaded"};
  if (prec == 2) {   // pair kernel phases
    const char* pn[] = {"start", "BD passed", "D loaded", "A stored", "BA done"};
    for (int g = 0; g < 2; ++g)
      for (int w = 0; w < 2; ++w) {
        printf("tile %d warp %s:", g, w ? "13" : "0 ");
        for (int p = 1; p <= 4; ++p) {
          std::vector<long long> d;
          for (int st = 200; st < 3000; ++st) d.push_back(tr[g][w][p][st] - tr[g][w][p - 1][st]);
          std::sort(d.begin(), d.end());
          printf("  %s-%s %lld", pn[p - 1], pn[p], d[d.size() / 2]);
        }
        std::vector<long long> d;
        for (int st = 200; st < 3000; ++st) d.push_back(tr[g][w][0][st + 1] - tr[g][w][0][st]);
        std::sort(d.begin(), d.end());
        printf("  | step %lld\n", d[d.size() / 2]);
      }
    return 0;
  }
  for (int g = 0; g < 2; ++g)
    for (int w = 0; w < 2; ++w) {
      printf("slot %d warp %s:", g, w ? "13" : "0 ");
      for (int p = 1; p <= 5; ++p) {
        std::vector<long long> d;
        for (int st = 200; st < 3000; ++st) d.push_back(tr[g][w][p][st] - tr[g][w][p - 1][st]);
        std::sort(d.begin(), d.end());
        printf("  %s-%s %lld", names[p - 1], names[p], d[d.size() / 2]);
      }
      std::vector<long long> d;
      for (int st = 200; st < 3000; ++st) d.push_back(tr[g][w][0][st + 1] - tr[g][w][0][st]);
      std::sort(d.begin(), d.end());
      printf("  | step %lld", d[d.size() / 2]);
      if (w == 0) {
        std::vector<long long> l, r;
        for (int st = 200; st < 3000; ++st) l.push_back(tr[g][0][6][st] - tr[g][0][2][st]), r.push_back(tr[g][0][7][st] - tr[g][0][3][st]);
        std::sort(l.begin(), l.end()); std::sort(r.begin(), r.end());
        printf("  | bar->locked %lld  issued->released %lld", l[l.size() / 2], r[r.size() / 2]);
      }
      printf("\n");
    }
  // absolute timeline of a few steps: events of both slots (warp 13 = non-issuer; issuer for 'issued')
  {
    const long long base = tr[0][1][0][1000];
    struct Ev { long long t; int g; int p; int st; };
    std::vector<Ev> ev;
    for (int g = 0; g < 2; ++g)
      for (int st = 990; st < 1010; ++st)
        for (int p = 0; p <= 5; ++p) {
          const long long t = tr[g][p == 3 ? 0 : 1][p][st] - base;
          if (t >= -500 && t < 9000) ev.push_back({t, g, p, st});
        }
    std::sort(ev.begin(), ev.end(), [](const Ev& x, const Ev& y) { return x.t < y.t; });
    for (auto& e : ev) printf("  t=%6lld slot %d step %d  %s\n", e.t, e.g, e.st, names[e.p]);
  }
  for (int g = 0; g < 2; ++g) {
    std::vector<long long> a1, a2;
    for (int st = 200; st < 3000; ++st) {
      a1.push_back(tr[g][0][7][st + 1] - tr[g][0][3][st]);   // issued (step st) -> poll success (next step)
      a2.push_back(tr[g][0][7][st + 1] - tr[g][0][6][st + 1]);
    }
    std::sort(a1.begin(), a1.end()); std::sort(a2.begin(), a2.end());
    printf("slot %d: issued -> MMA done seen %lld  (polling time %lld)\n", g, a1[a1.size() / 2], a2[a2.size() / 2]);
  }
  // cross-slot: when slot 1 issues relative to slot 0's D ready
  std::vector<long long> d;
  for (int st = 200; st < 3000; ++st) d.push_back(tr[1][0][3][st] - tr[0][0][4][st]);
  std::sort(d.begin(), d.end());
  printf("slot1 issued - slot0 D ready (same step index): %lld\n", d[d.size() / 2]);
  return 0;
}
