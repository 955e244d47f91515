// Microbenchmark of the per-sentence beam step kernel (step_kernels.cu), c2 shape
// (B = 30, K = 5, C = 148 partials per row, E = H = 500, L = 2), with phase stamps.
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <algorithm>
#include "../../paper_1805_11462_b200/csrc/step_kernels.cu"
using namespace onmt;
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); exit(1);} } while (0)
int main(int argc, char** argv) {
  const int rsplit = argc > 1 ? atoi(argv[1]) : 0;   // 1: the recurrent-split step's layer-1 cell
  const int rsdbg = argc > 2 ? atoi(argv[2]) : 0;
  CK(cudaMemcpyToSymbol(g_rs_dbg, &rsdbg, sizeof(int)));
  cudaStream_t st; CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  auto envi = [](const char* n, int d) { const char* v = getenv(n); return v ? atoi(v) : d; };
  const int B = envi("UB_B", 30), K = envi("UB_K", 5), R = B * K, NP = (R + 31) / 32 * 32, C = 148, E = 500,
            H = envi("UB_H", 500), L = 2, V = 50000, MAXLEN = 100;
  auto zalloc = [&](size_t bytes) { void* p; CK(cudaMalloc(&p, bytes)); CK(cudaMemset(p, 0, bytes)); return p; };
  // partials: random (m, s) and sorted random top-K lists, layout [r][C]
  std::vector<float2> hms((size_t)R * C); std::vector<float> htz((size_t)R * C * K); std::vector<int> hti((size_t)R * C * K);
  unsigned long long x = 1234567;
  auto rnd = [&]() { x ^= x << 13; x ^= x >> 7; x ^= x << 17; return (x >> 11) * (1.0 / 9007199254740992.0); };
  for (int r = 0; r < R; ++r) for (int p = 0; p < C; ++p) {
    const size_t i = (size_t)r * C + p;
    float top = 5.f + (float)rnd();
    hms[i] = make_float2(top, 10.f);
    for (int k = 0; k < K; ++k) { htz[i * K + k] = top - 0.3f * k - 0.1f * (float)rnd(); hti[i * K + k] = p * 338 + k; }
  }
  float2* ms = (float2*)zalloc(hms.size() * 8); float* tz = (float*)zalloc(htz.size() * 4); int* ti = (int*)zalloc(hti.size() * 4);
  CK(cudaMemcpy(ms, hms.data(), hms.size() * 8, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(tz, htz.data(), htz.size() * 4, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(ti, hti.data(), hti.size() * 4, cudaMemcpyHostToDevice));
  BeamState bs{};
  bs.cum = (double*)zalloc(2 * R * 8); bs.live = (int*)zalloc(2 * R * 4); bs.y = (int*)zalloc(R * 4);
  bs.prow = (int*)zalloc(R * 4); bs.done = (int*)zalloc(B * 4); bs.n_done = (int*)zalloc(4);
  bs.best_t = (int*)zalloc(B * 4); bs.best_r = (int*)zalloc(B * 4); bs.best_raw = (double*)zalloc(B * 8);
  bs.best_norm = (double*)zalloc(B * 8); bs.hist_parent = (int*)zalloc(MAXLEN * R * 4);
  bs.hist_token = (int*)zalloc(MAXLEN * R * 4); bs.hist_logp = (float*)zalloc(MAXLEN * R * 4);
  { std::vector<int> lv(2 * R, 1); CK(cudaMemcpy(bs.live, lv.data(), 2 * R * 4, cudaMemcpyHostToDevice)); }
  GatherArgs ga{};
  ga.emb_tgt = (float*)zalloc((size_t)V * E * 4); ga.E = E; ga.H = H; ga.L = L;
  ga.htilde = (float*)zalloc(NP * H * 4); ga.h = (float*)zalloc(L * NP * H * 4); ga.c = (float*)zalloc(L * NP * H * 4);
  ga.cg = (float*)zalloc(L * NP * H * 4); ga.rows_pad = NP;
  ga.x[0] = XOut{nullptr, (__nv_bfloat16*)zalloc(2 * NP * 1536 * 2), NP, 1536};
  ga.x[1] = XOut{nullptr, (__nv_bfloat16*)zalloc(2 * NP * 1024 * 2), NP, 1024};
  if (rsplit) {
    const int G = 2048;
    ga.rsplit = 1;
    ga.T = (float*)zalloc((size_t)V * G * 4);
    ga.P = (float*)zalloc((size_t)3 * NP * G * 4);
    ga.G = G;
    for (int l = 0; l < L; ++l) ga.bias[l] = (const float4*)zalloc(G * 4);
    ga.gb = (float*)zalloc((size_t)NP * G * 4);
    ga.c1_out = (float*)ga.c;
    ga.xh1[0] = XOut{nullptr, (__nv_bfloat16*)zalloc(2 * NP * 512 * 2), NP, 512}; ga.col_h1[0] = 0;
    ga.xh1[1] = XOut{nullptr, (__nv_bfloat16*)zalloc(2 * NP * 1536 * 2), NP, 1536}; ga.col_h1[1] = 512;
  }
  float* rl = (float*)zalloc(R * 4); float* rz = (float*)zalloc(R * K * 4); int* ri = (int*)zalloc(R * K * 4);
  unsigned long long* tr; CK(cudaMalloc(&tr, 4096 * 96)); CK(cudaMemcpyToSymbol(g_ktrace, &tr, sizeof(tr)));
  const int nsl = argc > 3 ? atoi(argv[3]) : 1;
  auto launch = [&]() { launch_beam_merge(ms, tz, ti, C, 1, C, B, K, 5, MAXLEN, 1.0, bs, ga, rl, rz, ri, StepCtl{nullptr, 0}, st, nsl, nullptr); };
  cudaGraph_t gr; cudaGraphExec_t ge;
  CK(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
  for (int i = 0; i < 20; ++i) launch();
  CK(cudaStreamEndCapture(st, &gr)); CK(cudaGraphInstantiate(&ge, gr, 0));
  for (int w = 0; w < 50; ++w) CK(cudaGraphLaunch(ge, st));
  CK(cudaStreamSynchronize(st));
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  CK(cudaEventRecord(a, st)); CK(cudaGraphLaunch(ge, st)); CK(cudaEventRecord(b, st)); CK(cudaStreamSynchronize(st));
  float ms_; cudaEventElapsedTime(&ms_, a, b);
  CK(cudaMemset(tr, 0, 4096 * 96)); CK(cudaGraphLaunch(ge, st)); launch(); CK(cudaStreamSynchronize(st));
  std::vector<unsigned long long> h(B * 12);
  CK(cudaMemcpy(h.data(), tr, B * 96, cudaMemcpyDeviceToHost));
  unsigned long long t0 = ~0ull; for (int c = 0; c < B; ++c) t0 = std::min(t0, h[c * 12]);
  double avg[12] = {0}, mx[12] = {0}; int cnt[12] = {0};
  for (int c = 0; c < B; ++c) for (int i = 0; i < 12; ++i) if (h[c * 12 + i]) {
    double d = (h[c * 12 + i] - t0) / 1e3; avg[i] += d; cnt[i]++; mx[i] = std::max(mx[i], d); }
  printf("beam_step rsplit=%d: %.2f us/launch (graph of 20)\n", rsplit, ms_ * 1000 / 20);
  const char* nm[12] = {"entry", "after pdl/done", "live/cum loaded", "rows reduced", "selected", "gather staged", "exit", "sc ready", "ranked", "owners done", "cell math done", "cell synced"};
  for (int i = 0; i < 12; ++i) if (cnt[i]) printf("   %-16s avg %7.2f  max %7.2f us (n=%d)\n", nm[i], avg[i] / cnt[i], mx[i], cnt[i]);
  {
    std::vector<unsigned long long> x(4);
    CK(cudaMemcpy(x.data(), tr + 34000, 32, cudaMemcpyDeviceToHost));
    const char* xn[4] = {"row0: partials loaded", "row0: theta done", "row0: lists merged", "row0: top-K out"};
    for (int i = 0; i < 4; ++i) if (x[i] > t0) printf("   %-24s %7.2f us\n", xn[i], (x[i] - t0) / 1e3);
  }
  return 0;
}
