// Teacher-forced scoring (PAPER.md P105-108: log p(Y | X) =
// sum_t log p(y_t | y_<t, X)): the decoder runs over the gold target tokens instead of
// the beam's selections, and the generator gathers the gold logit instead of a top-K.
//   teacher_gather_kernel  A5 with parent = self and y_{t-1} = the gold token (BOS at t = 1)
//   score_reduce_kernel    log p(gold) = z_gold - LSE from the generator's per-tile partials
//   score_row_kernel       (fp32 models) LSE and gold logit straight from a logits row
#include "common.cuh"

namespace onmt {

// x1 = [E_tgt[y]; h~; h_0], x_l = [.; h_l], c_prev_l = c_l for row r (no reordering)
__global__ void teacher_gather_kernel(const int* __restrict__ tgt, int T_max, int t, GatherArgs g) {
  pdl_trigger();
  pdl_wait();
  const int r = blockIdx.x;
  const int y = t == 1 ? 2 : __ldg(&tgt[(size_t)r * T_max + t - 2]);   // BOS = 2; pads (0) past the end
  const float* e = g.emb_tgt + (size_t)y * g.E;
  for (int c = threadIdx.x; c < g.E; c += blockDim.x) store_x(g.x[0], r, c, __ldg(&e[c]));
  for (int j = threadIdx.x; j < g.H; j += blockDim.x) {
    store_x(g.x[0], r, g.E + j, g.htilde[(size_t)r * g.H + j]);
    for (int l = 0; l < g.L; ++l) {
      const size_t src = ((size_t)l * g.rows_pad + r) * g.H + j;
      const float hv = g.h[src];
      if (l == 0) store_x(g.x[0], r, g.E + g.H + j, hv);
      else store_x(g.x[l], r, g.H + j, hv);
      g.cg[src] = g.c[src];
    }
  }
}

// one warp per generator row (t-1)*B + b: LSE over the n_vt tile partials, then
// log p = z_gold - LSE into out[b][t-1] (0 for rows past the sentence's length)
__global__ void score_reduce_kernel(const float2* __restrict__ ms, int n_vt, int rows_pad,
                                    const float* __restrict__ zgold, const int* __restrict__ gold, int B, int T_max,
                                    float* __restrict__ out) {
  pdl_trigger();
  pdl_wait();
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (warp >= B * T_max) return;
  const int row = warp, t1 = row / B, b = row % B;
  float m = -INFINITY, s = 0.f;
  for (int v = lane; v < n_vt; v += 32) {
    const float2 p = ms[(size_t)v * rows_pad + row];
    if (p.x == -INFINITY) continue;
    const float M = fmaxf(m, p.x);
    s = (m == -INFINITY ? 0.f : s * expf(m - M)) + p.y * expf(p.x - M);
    m = M;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const float m2 = __shfl_xor_sync(0xffffffffu, m, o), s2 = __shfl_xor_sync(0xffffffffu, s, o);
    const float M = fmaxf(m, m2);
    s = (m == -INFINITY ? 0.f : s * expf(m - M)) + (m2 == -INFINITY ? 0.f : s2 * expf(m2 - M));
    m = M;
  }
  if (lane == 0) out[(size_t)b * T_max + t1] = gold[row] >= 0 ? zgold[row] - (m + logf(s)) : 0.f;
}

// fp32 models: one CTA per row of a logits block [B][v_pad] (step t): LSE + gold logit
__global__ void score_row_kernel(const float* __restrict__ logits, int v_pad, const float* __restrict__ bias, int V,
                                 const int* __restrict__ gold, int B, int T_max, int t, float* __restrict__ out) {
  pdl_trigger();
  pdl_wait();
  const int b = blockIdx.x;
  const int gid = gold[(size_t)(t - 1) * B + b];
  const float* z = logits + (size_t)b * v_pad;
  float m = -INFINITY, s = 0.f;
  for (int v = threadIdx.x; v < V; v += blockDim.x) {
    const float x = z[v] + bias[v];
    if (x > m) { s = s * expf(m - x) + 1.f; m = x; }
    else s += expf(x - m);
  }
  __shared__ float sm_m[32], sm_s[32];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const float m2 = __shfl_xor_sync(0xffffffffu, m, o), s2 = __shfl_xor_sync(0xffffffffu, s, o);
    const float M = fmaxf(m, m2);
    s = (m == -INFINITY ? 0.f : s * expf(m - M)) + (m2 == -INFINITY ? 0.f : s2 * expf(m2 - M));
    m = M;
  }
  if (lane == 0) { sm_m[warp] = m; sm_s[warp] = s; }
  __syncthreads();
  if (threadIdx.x == 0) {
    float M = -INFINITY, S = 0.f;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
      const float m2 = sm_m[w], s2 = sm_s[w];
      const float Mx = fmaxf(M, m2);
      S = (M == -INFINITY ? 0.f : S * expf(M - Mx)) + (m2 == -INFINITY ? 0.f : s2 * expf(m2 - Mx));
      M = Mx;
    }
    out[(size_t)b * T_max + t - 1] = gid >= 0 ? (z[gid] + bias[gid]) - (M + logf(S)) : 0.f;
  }
}

void launch_teacher_gather(const int* tgt, int T_max, int t, int B, const GatherArgs& g, cudaStream_t st) {
  launch_pdl(teacher_gather_kernel, dim3(B), dim3(128), 0, st, tgt, T_max, t, g);
}
void launch_score_reduce(const float2* ms, int n_vt, int rows_pad, const float* zgold, const int* gold, int B,
                         int T_max, float* out, cudaStream_t st) {
  const int warps = B * T_max;
  launch_pdl(score_reduce_kernel, dim3((warps + 7) / 8), dim3(256), 0, st, ms, n_vt, rows_pad, zgold, gold, B, T_max,
             out);
}
void launch_score_row(const float* logits, int v_pad, const float* bias, int V, const int* gold, int B, int T_max,
                      int t, float* out, cudaStream_t st) {
  launch_pdl(score_row_kernel, dim3(B), dim3(256), 0, st, logits, v_pad, bias, V, gold, B, T_max, t, out);
}

}  // namespace onmt
