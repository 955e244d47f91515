// SIMT FFMA GEMM for fp32 models (and the bf16 debug backend): same contract as the
// tcgen05 kernel - split-K partials P[split][n][m] = sum_k W[m][k] X[n][k] - in fp32.
// fp32 parity (1e-5 on log-probs, BASELINE north_star) needs true fp32 products,
// which tf32 tensor cores do not give; the fp32 configuration (c1) is tiny and
// latency-bound, so FFMA is the right unit there.
#include "common.cuh"

namespace onmt {

template <typename TW>
__device__ __forceinline__ float ldw(const TW* p) { return static_cast<float>(*p); }
template <>
__device__ __forceinline__ float ldw<__nv_bfloat16>(const __nv_bfloat16* p) { return __bfloat162float(*p); }

// 64 (m) x 64 (n) output tile per 256-thread CTA, 4x4 per thread, K step 16.
template <typename TW>
__global__ void __launch_bounds__(256) simt_gemm_kernel(const TW* __restrict__ W, int m_pad, int k_pad,
                                                        const float* __restrict__ X, int n_rows_pad, int n_valid,
                                                        int k_per_split, float* __restrict__ out, StepCtl ctl) {
  pdl_trigger();
  pdl_wait();
  if (all_done(ctl)) return;
  __shared__ float Ws[16][64 + 4];
  __shared__ float Xs[16][64 + 4];
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  const int m0 = blockIdx.x * 64, n0 = blockIdx.y * 64;
  const int k_begin = blockIdx.z * k_per_split;
  int k_end = k_begin + k_per_split;
  if (k_end > k_pad) k_end = k_pad;
  float acc[4][4] = {};
  for (int k0 = k_begin; k0 < k_end; k0 += 16) {
    for (int e = threadIdx.x; e < 64 * 16; e += 256) {
      const int r = e >> 4, kk = e & 15;
      const int k = k0 + kk;
      const int m = m0 + r, n = n0 + r;
      Ws[kk][r] = (k < k_end && m < m_pad) ? ldw(W + (size_t)m * k_pad + k) : 0.f;
      Xs[kk][r] = (k < k_end && n < n_rows_pad) ? X[(size_t)n * k_pad + k] : 0.f;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < 16; ++kk) {
      float wv[4], xv[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) { wv[i] = Ws[kk][tx * 4 + i]; xv[i] = Xs[kk][ty * 4 + i]; }
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(wv[i], xv[j], acc[i][j]);
    }
    __syncthreads();
  }
  float* o = out + (size_t)blockIdx.z * n_rows_pad * m_pad;
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const int n = n0 + ty * 4 + j;
    if (n >= n_valid) continue;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int m = m0 + tx * 4 + i;
      if (m < m_pad) o[(size_t)n * m_pad + m] = acc[i][j];
    }
  }
}

template <int KMAX>
__global__ void gen_from_logits_kernel(const float* __restrict__ logits, int v_pad, GenOut g, StepCtl ctl) {
  pdl_trigger();
  pdl_wait();
  if (all_done(ctl)) return;
  const int vt = blockIdx.x;
  for (int r = threadIdx.x; r < g.rows_valid; r += blockDim.x) {
    float mx, sm, tz[KMAX];
    int ti[KMAX];
    scan_tile_column<KMAX>(logits + (size_t)r * v_pad + vt * kVTile, 1, vt * kVTile, g, mx, sm, tz, ti);
    write_gen_partial<KMAX>(g, vt, r, mx, sm, tz, ti);
  }
}

cudaError_t simt_gemm_partial(const void* W, bool w_bf16, int m_pad, int k_pad, const float* X, int n_rows_pad,
                              int n_valid, int splits, float* out, StepCtl ctl, cudaStream_t st) {
  int kps = (k_pad + splits - 1) / splits;
  kps = (kps + 15) / 16 * 16;
  dim3 grid((m_pad + 63) / 64, (n_rows_pad + 63) / 64, (k_pad + kps - 1) / kps);
  if (w_bf16)
    simt_gemm_kernel<__nv_bfloat16><<<grid, 256, 0, st>>>((const __nv_bfloat16*)W, m_pad, k_pad, X, n_rows_pad,
                                                          n_valid, kps, out, ctl);
  else
    simt_gemm_kernel<float><<<grid, 256, 0, st>>>((const float*)W, m_pad, k_pad, X, n_rows_pad, n_valid, kps, out,
                                                  ctl);
  return cudaGetLastError();
}

int simt_effective_splits(int k_pad, int splits) {
  int kps = (k_pad + splits - 1) / splits;
  kps = (kps + 15) / 16 * 16;
  return (k_pad + kps - 1) / kps;
}

cudaError_t simt_gen_partials(const float* logits, int v_pad, const GenOut& g, StepCtl ctl, cudaStream_t st) {
  dim3 grid((g.V + kVTile - 1) / kVTile);
  if (g.K <= 1) gen_from_logits_kernel<1><<<grid, 128, 0, st>>>(logits, v_pad, g, ctl);
  else if (g.K <= 2) gen_from_logits_kernel<2><<<grid, 128, 0, st>>>(logits, v_pad, g, ctl);
  else if (g.K <= 4) gen_from_logits_kernel<4><<<grid, 128, 0, st>>>(logits, v_pad, g, ctl);
  else if (g.K <= 8) gen_from_logits_kernel<8><<<grid, 128, 0, st>>>(logits, v_pad, g, ctl);
  else gen_from_logits_kernel<16><<<grid, 128, 0, st>>>(logits, v_pad, g, ctl);
  return cudaGetLastError();
}

}  // namespace onmt
