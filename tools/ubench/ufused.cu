// Microbenchmark of the cluster split-K fused GEMM (gemm_fused.cu) at the c2 decoder
// shapes, with per-CTA phase timestamps (ONMT_KTRACE).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -DONMT_KTRACE -I../../paper_1805_11462_b200/csrc \
//      -I../../include ufused.cu -lcuda -o ufused
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <algorithm>

#include "../../paper_1805_11462_b200/csrc/gemm_fused.cu"

using namespace onmt;
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); exit(1);} } while (0)

typedef CUresult (*PFN_encodeTiled_t)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                      const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                      CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
static CUtensorMap make_tmap(const void* base, int k_pad, int rows, int box_rows) {
  static PFN_encodeTiled_t fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
    fn = (PFN_encodeTiled_t)p;
  }
  CUtensorMap m;
  cuuint64_t dims[2] = {(cuuint64_t)k_pad, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)k_pad * 2};
  cuuint32_t box[2] = {64, (cuuint32_t)box_rows};
  cuuint32_t es[2] = {1, 1};
  CUresult r = fn(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, es,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) { printf("tmap fail\n"); exit(1); }
  return m;
}

int main() {
  cudaStream_t st;
  CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  const int H = 500, R = getenv("UF_R") ? atoi(getenv("UF_R")) : 150, NP = getenv("UF_NP") ? atoi(getenv("UF_NP")) : 160;
  struct Shape { const char* name; int M, K; bool tanh; int ns; bool fold; };
  // ns < NP: the recurrent-split step's layer-2 kernel (N-split groups of ns rows, whole K, per-row
  // gate bias gb); fold: the top layer's W_out[:, H:2H] h shares
  Shape shapes[] = {{"L1 gates 2000x1500", 4 * H, 3 * H, false, NP, false},
                    {"L2 gates 2000x1000 +fold", 4 * H, 2 * H, false, NP, true},
                    {"L2 gates 2000x1000", 4 * H, 2 * H, false, NP, false},
                    {"rsplit L2 2000x500 ns32 +gb", 4 * H, H, false, 32, false},
                    {"rsplit L2 2000x500 ns32 +gb +fold", 4 * H, H, false, 32, true},
                    {"W_out 500x1000 tanh", H, 2 * H, true, NP, false}};
  unsigned long long* tr;
  CK(cudaMalloc(&tr, 4096 * 96));
  CK(cudaMemcpyToSymbol(g_ktrace, &tr, sizeof(tr)));
  float *bias, *cg, *cout, *hout, *xo, *scratch;
  unsigned int* counters;
  CK(cudaMalloc(&scratch, 64 << 20));
  CK(cudaMalloc(&counters, 4096 * 4));
  CK(cudaMemset(counters, 0, 4096 * 4));
  __nv_bfloat16* xhl;
  CK(cudaMalloc(&bias, 4 * 4096 * 4));
  CK(cudaMalloc(&cg, NP * 1024 * 4));
  CK(cudaMalloc(&cout, NP * 1024 * 4));
  CK(cudaMalloc(&hout, NP * 1024 * 4));
  CK(cudaMalloc(&xo, NP * 2048 * 4));
  CK(cudaMalloc(&xhl, 2 * NP * 2048 * 2));
  CK(cudaMemset(bias, 0, 4 * 4096 * 4));
  float *gb, *woh_part;
  __nv_bfloat16* woh;
  CK(cudaMalloc(&gb, NP * 2048 * 4)); CK(cudaMemset(gb, 0, NP * 2048 * 4));
  CK(cudaMalloc(&woh_part, 16 * NP * H * 4));
  CK(cudaMalloc(&woh, 16 * fold_tile_bytes(H))); CK(cudaMemset(woh, 0, 16 * fold_tile_bytes(H)));
  for (int dbg = 0; dbg < 4; ++dbg)
  for (auto& sh : shapes) {
    g_fused_dbg = dbg;
    if (dbg && sh.tanh) continue;
    printf("[dbg mode %d] ", dbg);
    const int mp = (sh.M + 127) / 128 * 128, kp = (sh.K + 63) / 64 * 64;
    __nv_bfloat16 *W, *X;
    CK(cudaMalloc(&W, (size_t)mp * kp * 2));
    CK(cudaMalloc(&X, (size_t)2 * NP * kp * 2));
    CK(cudaMemset(W, 0, (size_t)mp * kp * 2));
    CK(cudaMemset(X, 0, (size_t)2 * NP * kp * 2));
    CUtensorMap tmW = make_tmap(W, kp, mp, 128), tmX = make_tmap(X, kp, 2 * NP, sh.ns);
    const bool rs = sh.ns < NP;
    XOut xd{nullptr, xhl, NP, 2048};
    CellDst dst{};
    dst.x[0] = xd; dst.col[0] = 0; dst.n = 1;
    auto launch = [&]() {
      cudaError_t err = sh.tanh ? tc_gemm_tanh(tmW, tmX, mp, NP, NP, R, kp / 64, H, hout, xd, scratch, counters, 148,
                                             StepCtl{nullptr, 0}, st)
                              : tc_gemm_cell(tmW, tmX, mp, NP, sh.ns, R, kp / 64, bias, cg, cout, hout, H, dst, scratch,
                                             counters, 148, StepCtl{nullptr, 0}, st, sh.fold ? woh : nullptr,
                                             sh.fold ? woh_part : nullptr, rs ? gb : nullptr, 2048);
      CK(err);
    };
    const int S = fused_split(sh.ns, NP, kp / 64, mp / 128, 148);
    const int grid = mp / 128 * (NP / sh.ns) * S;
    // graph of 50 launches
    cudaGraph_t g;
    cudaGraphExec_t ge;
    CK(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
    for (int i = 0; i < 50; ++i) launch();
    CK(cudaStreamEndCapture(st, &g));
    CK(cudaGraphInstantiate(&ge, g, 0));
    for (int w = 0; w < 400; ++w) CK(cudaGraphLaunch(ge, st));   // warm the clocks (~0.2 s)
    CK(cudaStreamSynchronize(st));
    cudaEvent_t a, b;
    cudaEventCreate(&a); cudaEventCreate(&b);
    CK(cudaEventRecord(a, st));
    CK(cudaGraphLaunch(ge, st));
    CK(cudaEventRecord(b, st));
    CK(cudaStreamSynchronize(st));
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    // single traced launch
    CK(cudaMemset(tr, 0, 4096 * 96));
    CK(cudaGraphLaunch(ge, st));
    launch();
    CK(cudaStreamSynchronize(st));
    std::vector<unsigned long long> h(grid * 12);
    CK(cudaMemcpy(h.data(), tr, grid * 96, cudaMemcpyDeviceToHost));
    unsigned long long t0 = ~0ull, t7 = 0;
    double avg[12] = {0}, mx[12] = {0};
    for (int c = 0; c < grid; ++c) t0 = std::min(t0, h[c * 12]);
    for (int c = 0; c < grid; ++c) {
      t7 = std::max(t7, h[c * 12 + 7]);
      for (int i = 0; i < 10; ++i) {
        double d = (double)(h[c * 12 + i] - t0) / 1e3;
        avg[i] += d / grid;
        mx[i] = std::max(mx[i], d);
      }
    }
    printf("%s: S=%d grid=%d  %.2f us/launch (graph of 50)  span %.2f us\n", sh.name, S, grid, ms * 1000 / 50,
           (t7 - t0) / 1e3);
    const char* nm[10] = {"entry", "after pdl_wait", "mma done", "partial stored", "tile complete", "partials in smem", "epilogue", "exit", "reduced", "reduced+sync"};
    for (int i = 0; i < 10; ++i) printf("   %-16s avg %7.2f  max %7.2f us\n", nm[i], avg[i], mx[i]);
    cudaFree(W); cudaFree(X);
  }
  return 0;
}
