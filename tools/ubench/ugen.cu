// Microbenchmark of the persistent generator step kernel (gen_step.cu), c2 shape
// (R = 150 rows, H = 500, V = 50000, K = 5), with per-CTA phase stamps; argv[1] = 1 adds the
// recurrent-split gate tiles (3 x 16 tiles of 128 x K 512 over an operand of 3 K blocks of 512).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -DONMT_KTRACE -I../../paper_1805_11462_b200/csrc \
//      -I../../include ugen.cu -lcuda -o ugen
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <algorithm>
#include "../../paper_1805_11462_b200/csrc/gen_step.cu"
#ifndef ONMT_KTRACE
__device__ unsigned long long* g_ktrace;   // (untraced build: the stamps below stay zero)
#endif
using namespace onmt;
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); exit(1);} } while (0)
typedef CUresult (*PFN_encodeTiled_t)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                      const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                      CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
static CUtensorMap make_tmap(const void* base, int k_pad, int rows, int box_rows) {
  static PFN_encodeTiled_t fn = nullptr;
  if (!fn) { void* p = nullptr; cudaDriverEntryPointQueryResult q;
    CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q)); fn = (PFN_encodeTiled_t)p; }
  CUtensorMap m;
  cuuint64_t dims[2] = {(cuuint64_t)k_pad, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)k_pad * 2};
  cuuint32_t box[2] = {64, (cuuint32_t)box_rows};
  cuuint32_t es[2] = {1, 1};
  if (fn(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
         CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) { printf("tmap\n"); exit(1); }
  return m;
}
int main(int argc, char** argv) {
  const int gates = argc > 1 ? atoi(argv[1]) : 0;
  g_gs_dbg = argc > 2 ? atoi(argv[2]) : 0;
  cudaStream_t st; CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  const int R = getenv("UG_R") ? atoi(getenv("UG_R")) : 150, NP = 160, KP = 512, V = 50000, VP = 50048,
            K = getenv("UG_K") ? atoi(getenv("UG_K")) : 5, C = 148;
  __nv_bfloat16 *W, *X; float* bias;
  const int XK = gates ? 3 * KP : KP;                        // operand width (gate tiles: [h~ | h1 | h2])
  CK(cudaMalloc(&W, (size_t)VP * KP * 2)); CK(cudaMalloc(&X, (size_t)2 * NP * XK * 2)); CK(cudaMalloc(&bias, VP * 4));
  {  // realistic values: W ~ U(-0.1, 0.1) bf16, activations tanh-like (hi plane; lo = 0), bias ~ U(-0.1, 0.1)
    std::vector<__nv_bfloat16> hw((size_t)VP * KP), hx((size_t)2 * NP * XK);
    std::vector<float> hb(VP);
    unsigned long long st_ = 88172645463325252ull;
    auto rnd = [&]() { st_ ^= st_ << 13; st_ ^= st_ >> 7; st_ ^= st_ << 17; return (st_ >> 11) * (1.0 / 9007199254740992.0); };
    for (size_t i = 0; i < hw.size(); ++i) hw[i] = __float2bfloat16((i % KP) < 500 ? (float)(0.2 * rnd() - 0.1) : 0.f);
    for (size_t i = 0; i < hx.size(); ++i) hx[i] = __float2bfloat16(i < (size_t)NP * XK && (i % KP) < 500 ? (float)tanh(3 * rnd() - 1.5) : 0.f);
    for (int i = 0; i < VP; ++i) hb[i] = i < V ? (float)(0.2 * rnd() - 0.1) : 0.f;
    CK(cudaMemcpy(W, hw.data(), hw.size() * 2, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(X, hx.data(), hx.size() * 2, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(bias, hb.data(), VP * 4, cudaMemcpyHostToDevice));
  }
  CUtensorMap tmW = make_tmap(W, KP, VP, 128), tmX = make_tmap(X, XK, 2 * NP, NP);
  const int G = 2048;
  __nv_bfloat16* Wg; float* gout;
  CK(cudaMalloc(&Wg, (size_t)3 * G * KP * 2)); CK(cudaMemset(Wg, 0, (size_t)3 * G * KP * 2));
  CK(cudaMalloc(&gout, (size_t)3 * NP * G * 4));
  CUtensorMap tmWg = make_tmap(Wg, KP, 3 * G, 128);
  GateTiles gt{};
  if (gates) gt = GateTiles{&tmWg, 3 * G / 128, G / 128, KP / 64, G, gout};
  float2* ms; float *tz, *rl, *rz; int *ti, *ri; unsigned int* gbar;
  CK(cudaMalloc(&ms, C * NP * 8)); CK(cudaMalloc(&tz, C * NP * K * 4)); CK(cudaMalloc(&ti, C * NP * K * 4));
  CK(cudaMalloc(&rl, R * 4)); CK(cudaMalloc(&rz, R * K * 4)); CK(cudaMalloc(&ri, R * K * 4));
  CK(cudaMalloc(&gbar, 64)); CK(cudaMemset(gbar, 0, 64));
  unsigned int* thr; CK(cudaMalloc(&thr, 2 * NP * 17 * 4)); CK(cudaMemset(thr, 0, 2 * NP * 17 * 4));
  unsigned long long* tr; CK(cudaMalloc(&tr, 4096 * 96)); CK(cudaMemcpyToSymbol(g_ktrace, &tr, sizeof(tr)));
  GenOut g{ms, tz, ti, bias, V, K, R, NP};
  const int MAXLEN = 100;
  int tstep = 2;  // alternate t: each launch clears the other threshold buffer, as in a decode
  auto launch = [&]() {
    tstep = tstep == 2 ? 3 : 2;
    CK(gen_step(tmW, tmX, VP / 128, NP, NP, KP / 64, 148, g, rl, rz, ri, tstep, thr, StepCtl{nullptr, 0}, st, gt, nullptr, 0, 0));
  };
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
  const int grid = C;
  std::vector<unsigned long long> h(grid * 12);
  CK(cudaMemcpy(h.data(), tr, grid * 96, cudaMemcpyDeviceToHost));
  unsigned long long t0 = ~0ull; for (int c = 0; c < grid; ++c) t0 = std::min(t0, h[c * 12]);
  double avg[12] = {0}, mx[12] = {0}; int cnt[12] = {0};
  for (int c = 0; c < grid; ++c) for (int i = 0; i < 12; ++i) if (h[c * 12 + i]) {
    double d = (h[c * 12 + i] - t0) / 1e3; avg[i] += d; cnt[i]++; mx[i] = std::max(mx[i], d); }
  printf("gen_step gates=%d dbg=%d: %.2f us/launch (graph of 20)\n", gates, g_gs_dbg, ms_ * 1000 / 20);
  (void)MAXLEN;
  const char* nm[12] = {"entry", "pdl_wait", "mma done (epi)", "phase A end", "scan0 start (w6)", "scan0 end (w6)", "stager: tile2 buf free", "first data (mma)", "batch scanned", "partial write", "stager: tile0 staged", "scan1 end (w6)"};
  for (int i = 0; i < 12; ++i) if (cnt[i]) printf("   %-16s avg %7.2f  max %7.2f us (n=%d)\n", nm[i], avg[i] / cnt[i], mx[i], cnt[i]);
  return 0;
}
