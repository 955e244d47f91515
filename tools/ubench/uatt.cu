// Microbenchmark of the cluster attention kernel (attention.cu) at the c2 shape (B=30,
// S_max=50, K=5, H=500, 'general' keys), graph of 50 launches + per-CTA phase stamps.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -DONMT_KTRACE -I../../paper_1805_11462_b200/csrc \
//      -I../../include uatt.cu -o uatt
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <algorithm>
#include "../../paper_1805_11462_b200/csrc/attention.cu"
using namespace onmt;
__global__ void calib(unsigned long long* out, float* sink) {
  unsigned long long g0, g1; long long c0, c1;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(g0));
  c0 = clock64();
  float x = threadIdx.x;
  for (int i = 0; i < 100000; ++i) x = fmaf(x, 0.999f, 0.001f);
  c1 = clock64();
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(g1));
  if (threadIdx.x == 0) { out[0] = g1 - g0; out[1] = c1 - c0; sink[0] = x; }
}
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); exit(1);} } while (0)
int main() {
  cudaStream_t st;
  CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  auto envi = [](const char* n, int d) { const char* v = getenv(n); return v ? atoi(v) : d; };
  const int B = envi("UATT_B", 30), S = envi("UATT_S", 50), K = envi("UATT_K", 5), H = envi("UATT_H", 500), KL = (H + 63) / 64 * 64;
  const int LO = envi("UATT_LO", 10), SPAN = envi("UATT_SPAN", 41);
  std::vector<int> lens(B);
  for (int b = 0; b < B; ++b) lens[b] = LO + (b * 37) % SPAN;
  int* dl; float *htop, *keys, *mem, *xf; __nv_bfloat16* xhl;
  CK(cudaMalloc(&dl, B * 4)); CK(cudaMemcpy(dl, lens.data(), B * 4, cudaMemcpyHostToDevice));
  CK(cudaMalloc(&htop, B * K * H * 4)); CK(cudaMalloc(&keys, (size_t)B * S * KL * 4)); CK(cudaMalloc(&mem, (size_t)B * S * H * 4));
  CK(cudaMemset(htop, 0, B * K * H * 4)); CK(cudaMemset(keys, 0, (size_t)B * S * KL * 4)); CK(cudaMemset(mem, 0, (size_t)B * S * H * 4));
  const int RP = (B * K + 31) / 32 * 32, XW = ((2 * H + 63) / 64) * 64;
  CK(cudaMalloc(&xhl, (size_t)2 * RP * XW * 2));
  unsigned long long* tr; CK(cudaMalloc(&tr, 8192 * 96)); CK(cudaMemcpyToSymbol(g_ktrace, &tr, sizeof(tr)));
  XOut xo{nullptr, xhl, RP, XW};
  // production configuration: folded W_out (values with ld 512, 16 top-layer tile shares)
  const bool fold = !getenv("UATT_PLAIN");
  float *wpart, *ht, *vals; __nv_bfloat16* xg;
  CK(cudaMalloc(&wpart, (size_t)16 * RP * H * 4)); CK(cudaMemset(wpart, 0, (size_t)16 * RP * H * 4));
  CK(cudaMalloc(&ht, (size_t)RP * H * 4)); CK(cudaMalloc(&xg, (size_t)2 * RP * XW * 2));
  CK(cudaMalloc(&vals, (size_t)B * S * KL * 4)); CK(cudaMemset(vals, 0, (size_t)B * S * KL * 4));
  AttFold fo{};
  if (fold) { fo.wpart = wpart; fo.n_wt = 16; fo.rows_pad = RP; fo.htilde = ht; fo.xg = XOut{nullptr, xg, RP, XW}; }
  auto launch = [&]() { CK(launch_attention(htop, keys, KL, fold ? vals : mem, fold ? KL : H, dl, B, S, H, K, xo, nullptr, 148,
                                            StepCtl{nullptr, 0}, st, fo)); };
  cudaGraph_t g; cudaGraphExec_t ge;
  CK(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
  for (int i = 0; i < 50; ++i) launch();
  CK(cudaStreamEndCapture(st, &g)); CK(cudaGraphInstantiate(&ge, g, 0));
  for (int w = 0; w < 400; ++w) CK(cudaGraphLaunch(ge, st));   // warm the clocks (~0.2 s)
  CK(cudaStreamSynchronize(st));
  cudaEvent_t a, b2; cudaEventCreate(&a); cudaEventCreate(&b2);
  CK(cudaEventRecord(a, st)); CK(cudaGraphLaunch(ge, st)); CK(cudaEventRecord(b2, st)); CK(cudaStreamSynchronize(st));
  float ms; cudaEventElapsedTime(&ms, a, b2);
  CK(cudaMemset(tr, 0, 8192 * 96)); CK(cudaGraphLaunch(ge, st)); launch(); CK(cudaStreamSynchronize(st));
  int nch = 148 / B; nch = nch > 8 ? 8 : nch; if (getenv("ONMT_ATT_NCH")) nch = atoi(getenv("ONMT_ATT_NCH"));
  const int grid = nch * B;
  std::vector<unsigned long long> h(grid * 12);
  CK(cudaMemcpy(h.data(), tr, grid * 96, cudaMemcpyDeviceToHost));
  unsigned long long t0 = ~0ull; for (int c = 0; c < grid; ++c) if (h[c * 12]) t0 = std::min(t0, h[c * 12]);
  double avg[12] = {0}, mx[12] = {0}; int cnt[12] = {0};
  for (int c = 0; c < grid; ++c) for (int i = 0; i < 9; ++i) if (h[c * 12 + i] >= t0 && h[c * 12]) {
    double d = (h[c * 12 + i] - t0) / 1e3; avg[i] += d; cnt[i]++; mx[i] = std::max(mx[i], d); }
  {
    unsigned long long* o; float* sk; CK(cudaMalloc(&o, 16)); CK(cudaMalloc(&sk, 4));
    calib<<<148, 32, 0, st>>>(o, sk); CK(cudaStreamSynchronize(st));
    unsigned long long hh[2]; CK(cudaMemcpy(hh, o, 16, cudaMemcpyDeviceToHost));
    printf("calib: 100k dependent FMA: %.1f us, %llu cycles -> %.0f MHz\n", hh[0] / 1e3, hh[1], hh[1] / (hh[0] / 1e3));
  }
  printf("attention B%d S%d K%d: %.2f us/launch (graph of 50)\n", B, S, K, ms * 1000 / 50);
  const char* nm[9] = {"entry", "prefetch issued", "pdl_wait", "sub0 staged", "scores", "parked", "cluster sync", "combined", "exit"};
  for (int i = 0; i < 9; ++i) printf("   %-16s avg %7.2f  max %7.2f us (n=%d)\n", nm[i], cnt[i] ? avg[i] / cnt[i] : 0, mx[i], cnt[i]);
  return 0;
}
