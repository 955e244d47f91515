// Device-side beam step (SURVEY §8(a) A10b + A5), shared by the stand-alone select/gather
// kernel (fp32 / SIMT path) and the persistent generator step kernel (gen_step.cu).
#pragma once
#include <math_constants.h>

#include "common.cuh"

namespace onmt {

// A10b + A5 for hypothesis row r, executed by one whole CTA (beam_device.cuh users):
// the K best (raw desc, slot asc, token asc) of sentence b's K x K row candidates with
// fp64 cumulative scores (O8); EOS / max_len banking, stop flag, histories (O9, O10) -
// computed redundantly by every CTA of the sentence from a few hundred bytes of state -
// then the CTA gathers column slice `slice` of `nslice` of row r's next-step decoder
// inputs (x1 = [E_tgt[y]; h~[p]; h_0[p]], x_l = [.; h_l[p]], c_l[p]).  The slice-0 CTA of
// row r writes slot r's beam state.  Row results (row_lse/z/i) may come from the same
// kernel (read with L2-coherent loads).
template <int KMAX>
__device__ __forceinline__ void select_gather_row(int r, int slice, int nslice, int R, const float* row_lse,
                                                  const float* row_z, const int* row_i, int K, int t, int max_len,
                                                  double lp, const BeamState& bs, const GatherArgs& ga) {
  const int b = r / K, kr = r % K;
  const int dn = __ldcg(&bs.done[b]);
  if (dn != 0 && dn < t) return;
  const int* __restrict__ live_in = bs.live + (size_t)(t & 1) * R;
  const double* __restrict__ cum_in = bs.cum + (size_t)(t & 1) * R;
  int* live_out = bs.live + (size_t)((t + 1) & 1) * R;
  double* cum_out = bs.cum + (size_t)((t + 1) & 1) * R;
  __shared__ int s_live[KMAX];
  __shared__ double s_cum[KMAX];
  __shared__ float s_lse[KMAX];
  __shared__ float s_z[KMAX][KMAX];
  __shared__ int s_id[KMAX][KMAX];
  __shared__ int s_prow, s_y, s_cont;
  if (threadIdx.x < K) {
    const int rr = b * K + threadIdx.x;
    s_live[threadIdx.x] = __ldcg(&live_in[rr]);
    s_cum[threadIdx.x] = __ldcg(&cum_in[rr]);
    s_lse[threadIdx.x] = __ldcg(&row_lse[rr]);
  }
  for (int i = threadIdx.x; i < K * K; i += blockDim.x) {
    s_z[i / K][i % K] = __ldcg(&row_z[(size_t)b * K * K + i]);
    s_id[i / K][i % K] = __ldcg(&row_i[(size_t)b * K * K + i]);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int head[KMAX];
    int sel_k[KMAX], sel_w[KMAX];
    double sel_s[KMAX];
    float sel_lp[KMAX];
    for (int k = 0; k < K; ++k) head[k] = 0;
    int n_sel = 0;
    for (int q = 0; q < K; ++q) {
      int bk = -1, bw = 0x7fffffff;
      double bsv = -CUDART_INF;
      for (int k = 0; k < K; ++k) {
        if (!s_live[k] || head[k] >= K) continue;
        const float z = s_z[k][head[k]];
        if (z == -INFINITY) continue;
        const double sc = s_cum[k] + ((double)z - (double)s_lse[k]);
        if (bk < 0 || sc > bsv) { bk = k; bsv = sc; bw = s_id[k][head[k]]; }
      }
      if (bk < 0) break;
      sel_k[n_sel] = bk; sel_w[n_sel] = bw; sel_s[n_sel] = bsv;
      sel_lp[n_sel] = (float)((double)s_z[bk][head[bk]] - (double)s_lse[bk]);
      ++n_sel;
      ++head[bk];
    }
    bool any_live = false;
    for (int q = 0; q < n_sel; ++q) any_live |= !(sel_w[q] == 3 || t == max_len);
    const bool stop = !any_live || t == max_len || (n_sel > 0 && sel_w[0] == 3);
    const bool mine_sel = kr < n_sel;
    const bool mine_live = mine_sel && !(sel_w[kr] == 3 || t == max_len);
    s_prow = mine_live ? b * K + sel_k[kr] : r;
    s_y = mine_live ? sel_w[kr] : 0;
    s_cont = !stop;
    if (slice == 0) {
      // this CTA owns slot kr of sentence b: slot state + history entry
      const size_t hb = (size_t)(t - 1) * (size_t)R + (size_t)r;
      live_out[r] = mine_live;
      cum_out[r] = mine_live ? sel_s[kr] : -CUDART_INF;
      bs.prow[r] = s_prow;
      bs.y[r] = s_y;
      bs.hist_parent[hb] = mine_sel ? sel_k[kr] : -1;
      bs.hist_token[hb] = mine_sel ? sel_w[kr] : 0;
      bs.hist_logp[hb] = mine_sel ? sel_lp[kr] : 0.f;
      if (bs.sel_parent) { bs.sel_parent[hb] = mine_sel ? sel_k[kr] : -1; bs.sel_score[hb] = mine_sel ? sel_s[kr] : -CUDART_INF; }
      if (kr == 0) {                                   // sentence-level banking and stop flag
        int bt = bs.best_t[b], br = bs.best_r[b];
        double braw = bs.best_raw[b], bnorm = bs.best_norm[b];
        for (int q = 0; q < n_sel; ++q) {
          if (sel_w[q] == 3 || t == max_len) {
            const double norm = sel_s[q] / lp;
            if (bt == 0 || norm > bnorm) { bt = t; br = q; braw = sel_s[q]; bnorm = norm; }
          }
        }
        bs.best_t[b] = bt; bs.best_r[b] = br; bs.best_raw[b] = braw; bs.best_norm[b] = bnorm;
        if (stop) { bs.done[b] = t; atomicAdd(bs.n_done, 1); }
      }
    }
  }
  __syncthreads();
  if (!s_cont) return;
  // ---- gather this CTA's column slice of row r (all loads first)
  const int p = s_prow, y = s_y;
  const int E = ga.E, H = ga.H, L = ga.L;
  const int e0 = (E * slice) / nslice, e1 = (E * (slice + 1)) / nslice;
  const int h0 = (H * slice) / nslice, h1 = (H * (slice + 1)) / nslice;
  const float* __restrict__ emb = ga.emb_tgt + (size_t)y * E;
  for (int c0 = e0 + threadIdx.x; c0 < e1; c0 += 2 * blockDim.x) {
    const int c1 = c0 + blockDim.x;
    const float v0 = __ldg(&emb[c0]);
    const float v1 = c1 < e1 ? __ldg(&emb[c1]) : 0.f;
    store_x(ga.x[0], r, c0, v0);
    if (c1 < e1) store_x(ga.x[0], r, c1, v1);
  }
  for (int j = h0 + threadIdx.x; j < h1; j += blockDim.x) {
    float hv[8], cv[8];
#pragma unroll
    for (int l = 0; l < 8; ++l)
      if (l < L) {
        hv[l] = __ldg(&ga.h[((size_t)l * ga.rows_pad + p) * H + j]);
        cv[l] = __ldg(&ga.c[((size_t)l * ga.rows_pad + p) * H + j]);
      }
    const float ht = __ldg(&ga.htilde[(size_t)p * H + j]);
    store_x(ga.x[0], r, E + j, ht);
#pragma unroll
    for (int l = 0; l < 8; ++l)
      if (l < L) {
        if (l == 0) store_x(ga.x[0], r, E + H + j, hv[l]);
        else store_x(ga.x[l], r, H + j, hv[l]);
        ga.cg[((size_t)l * ga.rows_pad + r) * H + j] = cv[l];
      }
  }
}

}  // namespace onmt
