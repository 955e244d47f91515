// Chip-wide global store throughput: G CTAs x 256 threads, each CTA writes BYTES with warp-
// coalesced 4-byte (or 16-byte) stores, st.global.cg (L2) - the fused cell kernel's fold-share
// write pattern (80 CTAs x 64 KB).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 ustore.cu -o ustore
#include <cstdio>
#include <cstdlib>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); exit(1);} } while (0)
__global__ void __launch_bounds__(1024) k_store(float* out, int per_cta_floats, int vec, unsigned long long* t) {
  unsigned long long t0, t1;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  float* o = out + (size_t)blockIdx.x * per_cta_floats;
  if (vec == 4) {
    float4* o4 = reinterpret_cast<float4*>(o);
    for (int i = threadIdx.x; i < per_cta_floats / 4; i += blockDim.x) __stcg(o4 + i, make_float4(1.f, 2.f, 3.f, (float)i));
  } else {
    for (int i = threadIdx.x; i < per_cta_floats; i += blockDim.x) __stcg(o + i, (float)i);
  }
  __syncthreads();
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
  if (threadIdx.x == 0) { t[2 * blockIdx.x] = t0; t[2 * blockIdx.x + 1] = t1; }
}
int main() {
  float* out; CK(cudaMalloc(&out, 256 << 20));
  unsigned long long* t; CK(cudaMalloc(&t, 4096 * 16));
  for (int nt : {256, 1024})
  for (int G : {1, 80, 148})
    for (int kb : {64, 256})
      for (int vec : {1, 4}) {
        const int pf = kb * 256;
        for (int w = 0; w < 3; ++w) { k_store<<<G, nt>>>(out, pf, vec, t); CK(cudaDeviceSynchronize()); }
        unsigned long long h[2 * 148];
        CK(cudaMemcpy(h, t, 2 * G * 8, cudaMemcpyDeviceToHost));
        unsigned long long a = ~0ull, b = 0; double avg = 0;
        for (int i = 0; i < G; ++i) { a = h[2 * i] < a ? h[2 * i] : a; b = h[2 * i + 1] > b ? h[2 * i + 1] : b; avg += (h[2 * i + 1] - h[2 * i]) / (double)G; }
        const double bytes = (double)G * kb * 1024;
        printf("threads %4d G=%3d %3d KB/CTA %s: per-CTA avg %.2f us (%.0f GB/s per SM), span %.2f us (%.2f TB/s chip)\n", nt, G, kb,
               vec == 4 ? "16B" : " 4B", avg / 1e3, kb * 1024 / avg, (b - a) / 1e3, bytes / (b - a) / 1e3);
      }
  return 0;
}
