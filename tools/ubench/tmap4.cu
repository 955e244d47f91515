// Does cuTensorMapEncodeTiled accept a 4D view {k_in, row, plane, k_block} of a [2][rows][k_pad]
// bf16 operand (strides not increasing)?  And does one 4D box land in the per-K-block layout?
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda.h>
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include "ptx.cuh"
using namespace onmt;
#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); exit(1);} } while (0)
typedef CUresult (*F)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                      const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                      CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
__global__ void k(const __grid_constant__ CUtensorMap tm, int n0, int rows, int nkb, unsigned short* out) {
  extern __shared__ __align__(1024) uint8_t sm_raw[];
  uint8_t* sm = sm_raw + ((1024u - (smem_u32(sm_raw) & 1023u)) & 1023u);
  __shared__ uint64_t bar;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1); fence_mbar_init();
    mbar_arrive_expect_tx(&bar, (uint32_t)nkb * 2 * rows * 128);
    asm volatile("cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], [%6];"
                 ::"r"(smem_u32(sm)), "l"(reinterpret_cast<uint64_t>(&tm)), "r"(0), "r"(n0), "r"(0), "r"(0), "r"(smem_u32(&bar)) : "memory");
    mbar_wait(&bar, 0);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < nkb * 2 * rows * 64; i += blockDim.x) out[i] = reinterpret_cast<unsigned short*>(sm)[i];
}
int main() {
  const int rows_pad = 160, k_pad = 512, ns = 32, nkb = 8, n0 = 64;
  std::vector<unsigned short> h((size_t)2 * rows_pad * k_pad);
  for (int p = 0; p < 2; ++p) for (int r = 0; r < rows_pad; ++r) for (int c = 0; c < k_pad; ++c)
    h[((size_t)p * rows_pad + r) * k_pad + c] = (unsigned short)((p * 7 + r * 13 + c * 3) & 0xffff);
  unsigned short* d; CK(cudaMalloc(&d, h.size() * 2)); CK(cudaMemcpy(d, h.data(), h.size() * 2, cudaMemcpyHostToDevice));
  void* fp = nullptr; cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &q));
  CUtensorMap m;
  cuuint64_t dims[4] = {64, (cuuint64_t)rows_pad, 2, (cuuint64_t)(k_pad / 64)};
  cuuint64_t strides[3] = {(cuuint64_t)k_pad * 2, (cuuint64_t)rows_pad * k_pad * 2, 128};
  cuuint32_t box[4] = {64, (cuuint32_t)ns, 2, (cuuint32_t)nkb};
  cuuint32_t es[4] = {1, 1, 1, 1};
  CUresult r = ((F)fp)(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, d, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                       CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encode 4D: %d\n", (int)r);
  if (r != CUDA_SUCCESS) return 0;
  unsigned short* o; CK(cudaMalloc(&o, (size_t)nkb * 2 * ns * 64 * 2));
  CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 80 * 1024));
  k<<<1, 256, 80 * 1024>>>(m, n0, ns, nkb, o); CK(cudaDeviceSynchronize());
  std::vector<unsigned short> g((size_t)nkb * 2 * ns * 64);
  CK(cudaMemcpy(g.data(), o, g.size() * 2, cudaMemcpyDeviceToHost));
  // expected smem: [kb][plane][row][64] with the 128-byte swizzle (16-byte chunk ^= row % 8)
  int bad = 0;
  for (int kb = 0; kb < nkb; ++kb) for (int p = 0; p < 2; ++p) for (int rr = 0; rr < ns; ++rr) for (int c = 0; c < 64; ++c) {
    const size_t tile = ((size_t)kb * 2 + p) * ns * 64;
    const int chunk = (c >> 3) ^ (rr & 7);
    const size_t off = tile + (size_t)rr * 64 + chunk * 8 + (c & 7);
    const unsigned short want = h[((size_t)p * rows_pad + n0 + rr) * k_pad + kb * 64 + c];
    if (g[off] != want && bad++ < 5) printf("mismatch kb %d p %d r %d c %d: %u vs %u\n", kb, p, rr, c, g[off], want);
  }
  printf("4D box layout [kb][plane][row][64] SW128: %s (%d bad)\n", bad ? "WRONG" : "OK", bad);
  return 0;
}
