// A7: Luong global attention for one decoder step (PAPER.md P119-122, P299-301; SURVEY
// §8(a) A7).  'general' scores are e_s = (W_in h) . m_s = h . (W_in^T m_s): the keys
// k_s = W_in^T m_s are computed once per batch after the encoder (one tcgen05 GEMM over
// every source position), so no per-step query GEMM exists; 'dot' uses k_s = m_s.
// a = softmax over s < S_b only (pads excluded), c_t = sum_s a_s m_s.
//
// One thread-block cluster per sentence b; cluster rank r owns source positions
// [r*CH, (r+1)*CH) (CH = ceil(S_max / nch), nch <= 8).  Each CTA
//   * prefetches its keys / memory rows with cp.async before griddepcontrol.wait (they are
//     constants of the translation), in sub-chunks of kSC positions, double-buffered;
//   * computes the K x kSC scores (one warp per position, lanes over H), and keeps an
//     online softmax per beam row (running max m_k, sum l_k) plus the unnormalised
//     context in registers (thread = columns j, all K rows);
//   * parks (m_k, l_k, ctx_k) in its shared memory; after a cluster barrier CTA r combines
//     column slice r over all nch chunks through distributed shared memory, in fixed chunk
//     order (deterministic), and writes the context into the W_out operand (columns [0, H)).
#include <cstdio>
#include <cstdlib>

#include "common.cuh"
#include "ptx.cuh"

namespace onmt {

constexpr int kSCMax = 16;       // positions per staged sub-chunk (16, or 8 for wide H)
constexpr int kAttThreads = 256;

__device__ __forceinline__ void cp_async_rows(float* dst, const float* src, int n) {
  const bool al = ((reinterpret_cast<uintptr_t>(src) | reinterpret_cast<uintptr_t>(dst)) & 15) == 0 && (n & 3) == 0;
  if (al) {
    for (int i = threadIdx.x; i < (n >> 2); i += blockDim.x)
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst + 4 * i)), "l"(src + 4 * i)
                   : "memory");
  } else {
    for (int i = threadIdx.x; i < n; i += blockDim.x)
      asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_u32(dst + i)), "l"(src + i) : "memory");
  }
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

__device__ __forceinline__ float ld_peer(const float* local, uint32_t peer) {
  float v;
  asm volatile("ld.shared::cluster.f32 %0, [%1];" : "=f"(v) : "r"(mapa_peer(smem_u32(local), peer)) : "memory");
  return v;
}
__device__ __forceinline__ float4 ld_peer4(const float* local, uint32_t peer) {
  float4 v;
  asm volatile("ld.shared::cluster.v4.f32 {%0, %1, %2, %3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "r"(mapa_peer(smem_u32(local), peer))
               : "memory");
  return v;
}

__device__ __forceinline__ float att_tanh(float x) {
  const float e = __expf(-2.f * fabsf(x));
  return copysignf(__fdividef(1.f - e, 1.f + e), x);
}

// Transposed butterfly: lane-partial sums of NV values (NV a power of two <= 32) reduced over
// the warp in log2(NV) halvings + the remaining pair sums; value index x ends on the lanes with
// xpose_index(lane) == x.  31 shuffles for 32 values instead of 5 per value.
template <int NV>
__device__ __forceinline__ float xpose_reduce(float (&v)[NV], int lane) {
#pragma unroll
  for (int h = NV / 2, o = 16; h >= 1; h /= 2, o /= 2) {
    const bool up = (lane & o) != 0;
#pragma unroll
    for (int i = 0; i < h; ++i) {
      const float send = up ? v[i] : v[i + h];
      const float keep = up ? v[i + h] : v[i];
      v[i] = keep + __shfl_xor_sync(0xffffffffu, send, o);
    }
  }
#pragma unroll
  for (int o = 16 / NV; o >= 1; o /= 2) v[0] += __shfl_xor_sync(0xffffffffu, v[0], o);
  return v[0];
}
template <int NV>
__device__ __forceinline__ int xpose_index(int lane) {
  int x = 0;
#pragma unroll
  for (int h = NV / 2, o = 16; h >= 1; h /= 2, o /= 2) x += (lane & o) ? h : 0;
  return x;
}
__host__ __device__ constexpr int pow2_at_least(int n) { return n <= 1 ? 1 : 2 * pow2_at_least((n + 1) / 2); }

template <int KMAX, int JPT>
__global__ void __launch_bounds__(kAttThreads)
attention_cluster_kernel(const float* __restrict__ htop, const float* __restrict__ keys, int key_ld,
                         const float* __restrict__ mem, int val_ld, const int* __restrict__ lens, int S_max, int H,
                         int K, int CH, int SC, XOut xo, const int* __restrict__ done, StepCtl ctl, AttFold fo) {
  KT(0);
  pdl_trigger();
  extern __shared__ __align__(16) float sh[];
  const int nch = gridDim.x;                      // cluster = the chunks of one sentence
  const uint32_t r = cluster_ctarank();
  const int b = blockIdx.y;
  const bool same = keys == mem;
  const int kl = same ? val_ld : key_ld;
  const int vl = val_ld;                          // value rows: m_s, or W_out[:, :H] m_s when folded
  const bool vec = (H & 3) == 0 && (kl & 3) == 0 && (vl & 3) == 0;
  auto r4 = [](size_t n) { return (n + 3) & ~(size_t)3; };
  // layout: q [K][H] (later: partial context) | m, l, scale [KMAX] | e [KMAX][16] |
  //         2 x (mem [SC][H], keys [SC][kl])
  float* q = sh;
  float* s_m = q + r4((size_t)K * H);              // (every region 16-byte aligned)
  float* s_l = s_m + kKMax;
  float* s_scale = s_l + kKMax;
  float* e = s_scale + kKMax;
  float* buf = e + kKMax * kSCMax;
  constexpr int KP = (KMAX + 3) & ~3;
  __shared__ __align__(16) float et[kSCMax * KP];   // softmax weights [position][row], rows >= K stay 0
  for (int i = threadIdx.x; i < kSCMax * KP; i += blockDim.x) et[i] = 0.f;
  const size_t mb = r4((size_t)SC * vl), kb = same ? 0 : r4((size_t)SC * kl);
  auto mbuf = [&](int i) { return buf + (size_t)(i & 1) * (mb + kb); };
  float* s_hp = buf + 2 * (mb + kb);                // folded W_out: the combine slice's tile shares
  float* s_esave = s_hp + fo.hp_floats;             // attention output: my chunk's raw scores [K][CH]
  // push combine (vec): every chunk stores its partial context slices into the owners' receive
  // buffers [source chunk][K][4 * wjm] and its (m, l) into every rank's s_rbm / s_rbl before the
  // cluster barrier; the combine then reads only local shared memory and no CTA reads a peer's
  // memory after the barrier (no trailing cluster barrier)
  // (measured: faster at c5 - 8 chunks, K = 10: 36 -> 28 us - slightly slower at c2 - 4 chunks, K = 5)
  const bool push = vec && fo.push;                // host plan: 8 chunks or K >= 8, and the buffer fits
  const int wjm = ((H >> 2) + nch - 1) / nch;
  float* rb = s_esave + (fo.att_out ? r4((size_t)K * CH) : 0);
  __shared__ float s_rbm[8 * KMAX], s_rbl[8 * KMAX];
  auto kbuf = [&](int i) { return same ? mbuf(i) : mbuf(i) + mb; };

  // source rows [s_beg, s_lim) of this chunk, prefetched before griddepcontrol.wait without
  // waiting for the length (rows past S_b are loaded but masked)
  const int s_beg = (int)r * CH;
  const int s_lim = min(S_max, s_beg + CH);
  const int nsub_max = s_lim > s_beg ? (s_lim - s_beg + SC - 1) / SC : 0;
  // sub-chunk staging: one bulk copy per operand (the chunk's rows are contiguous) completing on
  // the buffer's mbarrier - the TMA engine instead of 16-byte cp.async per thread, which bounded
  // the loop at ~5 us per sub-chunk for 1000-wide rows; cp.async when the rows are not 16-byte
  // aligned
  const bool bulk = vec && ((reinterpret_cast<uintptr_t>(mem) | reinterpret_cast<uintptr_t>(keys)) & 15) == 0;
  __shared__ __align__(8) uint64_t s_sbar[2];
  if (bulk && threadIdx.x == 0) { mbar_init(&s_sbar[0], 1); mbar_init(&s_sbar[1], 1); fence_mbar_init(); }
  if (bulk) __syncthreads();
  int n_staged = 0;                                // bulk stages issued (waited before exit)
  auto stage = [&](int i) {
    const int s0 = s_beg + i * SC;
    const int ns = min(SC, s_lim - s0);
    if (bulk) {
      if (threadIdx.x == 0) {
        const uint32_t mbytes = (uint32_t)ns * vl * 4, kbytes = same ? 0u : (uint32_t)ns * key_ld * 4;
        mbar_arrive_expect_tx(&s_sbar[i & 1], mbytes + kbytes);
        bulk_g2s(mbuf(i), mem + ((size_t)b * S_max + s0) * vl, mbytes, &s_sbar[i & 1]);
        if (!same) bulk_g2s(kbuf(i), keys + ((size_t)b * S_max + s0) * key_ld, kbytes, &s_sbar[i & 1]);
      }
      n_staged = i + 1;
      return;
    }
    cp_async_rows(mbuf(i), mem + ((size_t)b * S_max + s0) * vl, ns * vl);
    if (!same) cp_async_rows(kbuf(i), keys + ((size_t)b * S_max + s0) * key_ld, ns * key_ld);
    cp_async_commit();
  };
  auto stage_wait = [&](int i) { mbar_wait(&s_sbar[i & 1], (uint32_t)((i >> 1) & 1)); };
  if (nsub_max > 0) stage(0);
  if (nsub_max > 1) stage(1);
  KT(1);
  if (push) cluster_arrive_relaxed();              // (waited for before the first DSMEM store)
  pdl_wait();                                      // h_top, done flags of this step now visible
  const bool quit = all_done(ctl) || (done && done[b]);   // uniform over the cluster
  if (quit) {
    cp_async_wait<0>();
    if (bulk) for (int i = 0; i < n_staged; ++i) stage_wait(i);   // (no copy may land after exit)
    if (push) cluster_wait();                      // (complete the barrier phase opened above)
    return;
  }
  // queries: the K beam rows of sentence b - in registers for small K (each lane's 4 float4
  // columns of every row, reused by every position), else staged in shared memory
  // (5 < K <= 10: each half of the warps holds half of the rows, QSPLIT)
  constexpr bool QREG = KMAX <= 5 && JPT == 2;
  constexpr bool QSPLIT = KMAX > 5 && KMAX <= 10 && JPT == 2;
  constexpr int QR = QREG ? KMAX : QSPLIT ? (KMAX + 1) / 2 : 1;   // rows held per warp
  const int qrow0 = QSPLIT ? (threadIdx.x >> 7) * QR : 0;         // first row of this warp (half)
  float4 qr[QR][4];
  if ((QREG || QSPLIT) && vec) {
#pragma unroll
    for (int kk = 0; kk < QR; ++kk)
#pragma unroll
      for (int it = 0; it < 4; ++it) {
        const int j = 4 * (threadIdx.x & 31) + 128 * it, k = qrow0 + kk;
        qr[kk][it] = (k < K && j < H) ? __ldg(reinterpret_cast<const float4*>(htop + ((size_t)b * K + k) * H + j))
                                      : make_float4(0.f, 0.f, 0.f, 0.f);
      }
  } else {
    cp_async_rows(q, htop + (size_t)b * K * H, K * H);
  }
  cp_async_commit();
  // folded W_out: prefetch this CTA's combine slice of the top layer's W_out h shares
  // [tile][k][column] (produced by the previous kernel) - they land while the scores run
  const bool hpref = fo.wpart && fo.pref && vec;
  const int cj0 = (int)((long long)(H >> 2) * r / nch), cwj = (int)((long long)(H >> 2) * (r + 1) / nch) - cj0;
  if (hpref) {
    const int nit = K * cwj;
    for (int idx = threadIdx.x; idx < fo.n_wt * nit; idx += blockDim.x) {
      const int t = idx / nit, it = idx % nit;
      const int k = it / cwj, j = 4 * (cj0 + it % cwj);
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(s_hp + 4 * (size_t)idx)),
                   "l"(fo.wpart + ((size_t)t * fo.rows_pad + b * K + k) * H + j)
                   : "memory");
    }
    cp_async_commit();
  }
  const int L = lens[b];
  const int s_end = min(L, s_lim);
  const int nsub = s_end > s_beg ? (s_end - s_beg + SC - 1) / SC : 0;
  if (threadIdx.x < KMAX) { s_m[threadIdx.x] = -INFINITY; s_l[threadIdx.x] = 0.f; }
  KT(2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  float acc[KMAX][JPT];
#pragma unroll
  for (int k = 0; k < KMAX; ++k)
#pragma unroll
    for (int u = 0; u < JPT; ++u) acc[k][u] = 0.f;

  for (int i = 0; i < nsub; ++i) {
    if (bulk) {
      if (i == 0) {                                          // q (the W_out shares may stay in flight)
        if (hpref) cp_async_wait<1>();
        else cp_async_wait<0>();
      }
      stage_wait(i);
    } else if (i + 1 >= nsub_max) cp_async_wait<0>();
    else if (i == 0) {                                       // (iteration 0 also needs q; the
      if (hpref) cp_async_wait<1>();                         //  W_out shares may stay in flight)
      else cp_async_wait<0>();
    }
    else cp_async_wait<1>();
    __syncthreads();
    if (i == 0) KT(3);
    const int s0 = s_beg + i * SC;
    const int ns = min(SC, s_end - s0);
    const float* ms = mbuf(i);
    const float* ks = kbuf(i);
    // ---- scores: warp w -> positions w and w + 8 (they share the q loads)
    if (QSPLIT && vec) {
      // row half h = warp / 4 holds rows [h*QR, h*QR + QR); its 4 warps take the position
      // pairs (w, w + 8) and (w + 4, w + 12), w = warp % 4
#pragma unroll 1
      for (int pp = 0; pp < 2; ++pp) {
        const int pa = (warp & 3) + 4 * pp, pb = pa + 8;
        const bool ha = pa < ns, hb = pb < ns;
        if (!ha) continue;
        float da[QR], db[QR];
#pragma unroll
        for (int kk = 0; kk < QR; ++kk) { da[kk] = 0.f; db[kk] = 0.f; }
        const float* kra = ks + (size_t)pa * kl;
        const float* krb = ks + (size_t)(hb ? pb : pa) * kl;
#pragma unroll
        for (int it = 0; it < 4; ++it) {
          const int j = 4 * lane + 128 * it;
          if (j >= H) break;
          const float4 ka = *reinterpret_cast<const float4*>(kra + j);
          const float4 kbv = *reinterpret_cast<const float4*>(krb + j);
#pragma unroll
          for (int kk = 0; kk < QR; ++kk) {
            const float4 qv = qr[kk][it];
            da[kk] = fmaf(qv.x, ka.x, fmaf(qv.y, ka.y, fmaf(qv.z, ka.z, fmaf(qv.w, ka.w, da[kk]))));
            db[kk] = fmaf(qv.x, kbv.x, fmaf(qv.y, kbv.y, fmaf(qv.z, kbv.z, fmaf(qv.w, kbv.w, db[kk]))));
          }
        }
        constexpr int NV = pow2_at_least(2 * QR);
        float v[NV];
#pragma unroll
        for (int x = 0; x < NV; ++x) v[x] = x < QR ? da[x] : x < 2 * QR ? db[x - QR] : 0.f;
        const float sum = xpose_reduce<NV>(v, lane);
        const int x = xpose_index<NV>(lane);
        if ((lane & (32 / NV - 1)) == 0 && x < 2 * QR) {
          const int k = qrow0 + (x < QR ? x : x - QR);
          const int p = x < QR ? pa : pb;
          if (k < K && (x < QR || hb)) {
            e[k * kSCMax + p] = sum;
            if (fo.att_out) s_esave[k * CH + (s0 - s_beg) + p] = sum;
          }
        }
      }
    } else {
      const int pa = warp, pb = warp + 8;
      const bool ha = pa < ns, hb = pb < ns;
      if (ha) {
        float da[KMAX], db[KMAX];
#pragma unroll
        for (int k = 0; k < KMAX; ++k) { da[k] = 0.f; db[k] = 0.f; }
        const float* kra = ks + (size_t)pa * kl;
        const float* krb = ks + (size_t)(hb ? pb : pa) * kl;
        if (QREG && vec) {
#pragma unroll
          for (int it = 0; it < 4; ++it) {
            const int j = 4 * lane + 128 * it;
            if (j >= H) break;
            const float4 ka = *reinterpret_cast<const float4*>(kra + j);
            const float4 kbv = *reinterpret_cast<const float4*>(krb + j);
#pragma unroll
            for (int k = 0; k < KMAX; ++k) {
              const float4 qv = qr[QREG ? k : 0][it];
              da[k] = fmaf(qv.x, ka.x, fmaf(qv.y, ka.y, fmaf(qv.z, ka.z, fmaf(qv.w, ka.w, da[k]))));
              db[k] = fmaf(qv.x, kbv.x, fmaf(qv.y, kbv.y, fmaf(qv.z, kbv.z, fmaf(qv.w, kbv.w, db[k]))));
            }
          }
        } else if (vec) {
          for (int j = 4 * lane; j < H; j += 128) {
            const float4 ka = *reinterpret_cast<const float4*>(kra + j);
            const float4 kbv = *reinterpret_cast<const float4*>(krb + j);
#pragma unroll
            for (int k = 0; k < KMAX; ++k)
              if (k < K) {
                const float4 qv = *reinterpret_cast<const float4*>(q + (size_t)k * H + j);
                da[k] = fmaf(qv.x, ka.x, fmaf(qv.y, ka.y, fmaf(qv.z, ka.z, fmaf(qv.w, ka.w, da[k]))));
                db[k] = fmaf(qv.x, kbv.x, fmaf(qv.y, kbv.y, fmaf(qv.z, kbv.z, fmaf(qv.w, kbv.w, db[k]))));
              }
          }
        } else {
          for (int j = lane; j < H; j += 32) {
            const float ka = kra[j], kbv = krb[j];
#pragma unroll
            for (int k = 0; k < KMAX; ++k)
              if (k < K) {
                const float qv = q[(size_t)k * H + j];
                da[k] = fmaf(qv, ka, da[k]);
                db[k] = fmaf(qv, kbv, db[k]);
              }
          }
        }
        // warp sums of the 2 x KMAX dot products (transposed butterfly)
        constexpr int NV = pow2_at_least(2 * KMAX);
        float v[NV];
#pragma unroll
        for (int x = 0; x < NV; ++x) v[x] = x < KMAX ? da[x] : x < 2 * KMAX ? db[x - KMAX] : 0.f;
        const float sum = xpose_reduce<NV>(v, lane);
        const int x = xpose_index<NV>(lane);
        if ((lane & (32 / NV - 1)) == 0 && x < 2 * KMAX) {
          const int k = x < KMAX ? x : x - KMAX;
          const int p = x < KMAX ? pa : pb;
          if (k < K && (x < KMAX || hb)) {
            e[k * kSCMax + p] = sum;
            if (fo.att_out) s_esave[k * CH + (s0 - s_beg) + p] = sum;
          }
        }
      }
    }
    __syncthreads();
    if (i == 0) KT(4);
    // ---- online softmax per beam row (warp k, lanes = positions)
    for (int k = warp; k < K; k += kAttThreads / 32) {
      const float v = lane < ns ? e[k * kSCMax + lane] : -INFINITY;
      float mx = v;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
      const float mo = s_m[k];
      const float mn = fmaxf(mo, mx);
      const float w = lane < ns ? expf(v - mn) : 0.f;
      float sum = w;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
      if (lane < kSCMax) et[lane * KP + k] = w;   // (transposed: the context reads 4 rows at once)
      if (lane == 0) {
        const float sc = mo == -INFINITY ? 0.f : expf(mo - mn);
        s_scale[k] = sc;
        s_l[k] = s_l[k] * sc + sum;
        s_m[k] = mn;
      }
    }
    __syncthreads();
    // ---- context: thread owns columns j = tid + u*256
#pragma unroll
    for (int u = 0; u < JPT; ++u) {
      const int j = threadIdx.x + u * kAttThreads;
      if (j >= H) continue;
#pragma unroll
      for (int k = 0; k < KMAX; ++k)
        if (k < K) acc[k][u] *= s_scale[k];
      for (int s = 0; s < ns; ++s) {
        const float mv = ms[(size_t)s * vl + j];
        const float4* ev = reinterpret_cast<const float4*>(et + s * KP);
#pragma unroll
        for (int k4 = 0; k4 < KP / 4; ++k4) {              // (rows >= K hold weight 0)
          const float4 w = ev[k4];
          if (4 * k4 < KMAX) acc[4 * k4][u] = fmaf(w.x, mv, acc[4 * k4][u]);
          if (4 * k4 + 1 < KMAX) acc[4 * k4 + 1][u] = fmaf(w.y, mv, acc[4 * k4 + 1][u]);
          if (4 * k4 + 2 < KMAX) acc[4 * k4 + 2][u] = fmaf(w.z, mv, acc[4 * k4 + 2][u]);
          if (4 * k4 + 3 < KMAX) acc[4 * k4 + 3][u] = fmaf(w.w, mv, acc[4 * k4 + 3][u]);
        }
      }
    }
    __syncthreads();                               // buffer (i & 1) free for sub-chunk i + 2
    if (i + 2 < nsub_max) stage(i + 2);
  }
  if (hpref) cp_async_wait<1>();                   // (q, and prefetches past S_b; the W_out shares
  else cp_async_wait<0>();                         //  are waited for only by the combine)
  if (bulk) for (int i = nsub; i < n_staged; ++i) stage_wait(i);   // (stages past S_b)
  __syncthreads();
  if (push) {
    // ---- push my unnormalised partial context: column j goes to the chunk that owns it
    cluster_wait();                                // every peer CTA has started (DSMEM targets exist)
    const int H4 = H >> 2;
#pragma unroll
    for (int u = 0; u < JPT; ++u) {
      const int j = threadIdx.x + u * kAttThreads;
      if (j >= H) continue;
      const int j4 = j >> 2;
      int o = nch - 1;
      while (o > 0 && (int)((long long)H4 * o / nch) > j4) --o;
      const int j0o = (int)((long long)H4 * o / nch);
      const uint32_t base = mapa_peer(smem_u32(rb + ((size_t)r * K) * 4 * wjm + (j - 4 * j0o)), (uint32_t)o);
#pragma unroll
      for (int k = 0; k < KMAX; ++k)
        if (k < K) st_cluster_b32(base + (uint32_t)(k * 4 * wjm) * 4u, __float_as_uint(acc[k][u]));
    }
    if (threadIdx.x < K) {
      const int k = threadIdx.x;
      for (int p = 0; p < nch; ++p) {
        st_cluster_b32(mapa_peer(smem_u32(s_rbm + r * KMAX + k), (uint32_t)p), __float_as_uint(s_m[k]));
        st_cluster_b32(mapa_peer(smem_u32(s_rbl + r * KMAX + k), (uint32_t)p), __float_as_uint(s_l[k]));
      }
    }
  } else {
    // ---- park the unnormalised partial context in q's place (q is no longer read)
#pragma unroll
    for (int u = 0; u < JPT; ++u) {
      const int j = threadIdx.x + u * kAttThreads;
      if (j >= H) continue;
#pragma unroll
      for (int k = 0; k < KMAX; ++k)
        if (k < K) q[(size_t)k * H + j] = acc[k][u];
    }
  }
  KT(5);
  cluster_arrive();
  cluster_wait();
  KT(6);
  // ---- combine: CTA r finalises columns [j0, j1) of every beam row over all chunks
  float* coef = e;                                 // [8][KMAX] (e is free now)
  if (threadIdx.x < K) {
    const int k = threadIdx.x;
    float mp[8], lp[8];
    if (push) {
#pragma unroll
      for (int p = 0; p < 8; ++p) {
        mp[p] = p < nch ? s_rbm[p * KMAX + k] : -INFINITY;
        lp[p] = p < nch ? s_rbl[p * KMAX + k] : 0.f;
      }
    } else {
#pragma unroll
      for (int p = 0; p < 8; ++p) {
        mp[p] = p < nch ? ld_peer(s_m + k, p) : -INFINITY;
        lp[p] = p < nch ? ld_peer(s_l + k, p) : 0.f;
      }
    }
    float M = -INFINITY;
#pragma unroll
    for (int p = 0; p < 8; ++p) M = fmaxf(M, mp[p]);
    float Ls = 0.f;
#pragma unroll
    for (int p = 0; p < 8; ++p) {
      const float w = mp[p] == -INFINITY ? 0.f : expf(mp[p] - M);
      mp[p] = w;
      Ls += lp[p] * w;
    }
    const float inv = 1.f / Ls;
#pragma unroll
    for (int p = 0; p < 8; ++p) coef[p * KMAX + k] = mp[p] * inv;
  }
  if (hpref) cp_async_wait<0>();                   // my prefetched W_out shares (and any stage)
  __syncthreads();
  if (fo.att_out) {
    // normalised weights of my chunk (coverage / unknown replacement, S436-448):
    // a_s = exp(e_s - m_r) * exp(m_r - M) / l  (zero at padded positions)
    for (int i = threadIdx.x; i < K * (s_lim - s_beg); i += blockDim.x) {
      const int k = i / (s_lim - s_beg), s = s_beg + i % (s_lim - s_beg);
      const float a = s < L ? expf(s_esave[k * CH + (s - s_beg)] - s_m[k]) * coef[r * KMAX + k] : 0.f;
      fo.att_out[((size_t)b * K + k) * S_max + s] = a;
    }
  }
  if (vec) {
    const int H4 = H >> 2;
    const int j0 = (int)((long long)H4 * r / nch), j1 = (int)((long long)H4 * (r + 1) / nch);
    const int wj = j1 - j0;
    for (int it = threadIdx.x; it < K * wj; it += blockDim.x) {
      const int k = it / wj, j = 4 * (j0 + it % wj);
      float4 v[8];
      if (push) {                                  // (separate loops: the DSMEM loads stay back to back)
#pragma unroll
        for (int p = 0; p < 8; ++p)
          v[p] = p < nch ? *reinterpret_cast<const float4*>(rb + ((size_t)p * K + k) * 4 * wjm + (j - 4 * j0))
                         : make_float4(0.f, 0.f, 0.f, 0.f);
      } else {
#pragma unroll
        for (int p = 0; p < 8; ++p) v[p] = p < nch ? ld_peer4(q + (size_t)k * H + j, p) : make_float4(0.f, 0.f, 0.f, 0.f);
      }
      float4 c = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
      for (int p = 0; p < 8; ++p) {
        const float w = coef[p * KMAX + k];
        c.x = fmaf(w, v[p].x, c.x); c.y = fmaf(w, v[p].y, c.y); c.z = fmaf(w, v[p].z, c.z); c.w = fmaf(w, v[p].w, c.w);
      }
      const int row = b * K + k;
      if (fo.wpart) {
        // folded W_out: c = W_out[:, :H] c_t (values were projected); add the top cell layer's
        // W_out[:, H:2H] h_t shares (fixed tile order) and finish h~ = tanh(.)
        float4 hs = make_float4(0.f, 0.f, 0.f, 0.f);
        if (hpref) {                                               // prefetched (fixed tile order)
          for (int t = 0; t < fo.n_wt; ++t) {
            const float4 pv = *reinterpret_cast<const float4*>(s_hp + 4 * ((size_t)t * K * wj + it));
            hs.x += pv.x; hs.y += pv.y; hs.z += pv.z; hs.w += pv.w;
          }
        } else
        for (int t0 = 0; t0 < fo.n_wt; t0 += 8) {                 // 8 loads in flight, fixed order
          float4 pv[8];
#pragma unroll
          for (int u = 0; u < 8; ++u)
            pv[u] = t0 + u < fo.n_wt ? __ldcg(reinterpret_cast<const float4*>(fo.wpart + ((size_t)(t0 + u) * fo.rows_pad + row) * H + j))
                                     : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
          for (int u = 0; u < 8; ++u) { hs.x += pv[u].x; hs.y += pv[u].y; hs.z += pv[u].z; hs.w += pv[u].w; }
        }
        const float4 ht = make_float4(att_tanh(c.x + hs.x), att_tanh(c.y + hs.y), att_tanh(c.z + hs.z), att_tanh(c.w + hs.w));
        *reinterpret_cast<float4*>(fo.htilde + (size_t)row * H + j) = ht;
        store_x4(fo.xg, row, j, ht);                               // (8-byte hi / lo stores)
      } else {
        store_x4(xo, row, j, c);
      }
    }
  } else {
    const int j0 = (int)((long long)H * r / nch), j1 = (int)((long long)H * (r + 1) / nch);
    const int wj = j1 - j0;
    for (int it = threadIdx.x; it < K * wj; it += blockDim.x) {
      const int k = it / wj, j = j0 + it % wj;
      float v[8];
#pragma unroll
      for (int p = 0; p < 8; ++p) v[p] = p < nch ? ld_peer(q + (size_t)k * H + j, p) : 0.f;
      float c = 0.f;
#pragma unroll
      for (int p = 0; p < 8; ++p) c = fmaf(coef[p * KMAX + k], v[p], c);
      const int row = b * K + k;
      if (fo.wpart) {
        float hs = 0.f;
        for (int t0 = 0; t0 < fo.n_wt; t0 += 8) {
          float pv[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) pv[u] = t0 + u < fo.n_wt ? __ldcg(fo.wpart + ((size_t)(t0 + u) * fo.rows_pad + row) * H + j) : 0.f;
#pragma unroll
          for (int u = 0; u < 8; ++u) hs += pv[u];
        }
        const float ht = att_tanh(c + hs);
        fo.htilde[(size_t)row * H + j] = ht;
        store_x(fo.xg, row, j, ht);
      } else {
        store_x(xo, row, j, c);
      }
    }
  }
  KT(7);
  if (!push) {
    cluster_arrive();                              // peers may still be reading my partial
    cluster_wait();
  }
  KT(8);
}

// chunks per sentence: fill the SMs with one wave of clusters (<= 8 CTAs, >= 4 positions each)
static int att_nch(int B, int S_max, int num_sms) {
  if (const char* e = std::getenv("ONMT_ATT_NCH")) return std::atoi(e);   // (tuning experiments)
  int nch = num_sms / (B > 0 ? B : 1);
  nch = nch > 8 ? 8 : nch < 1 ? 1 : nch;
  const int pos_cap = (S_max + 3) / 4;
  return nch > pos_cap ? (pos_cap < 1 ? 1 : pos_cap) : nch;
}

template <int KMAX, int JPT>
static cudaError_t launch_att(dim3 grid, int nch, size_t smem, cudaStream_t st, const float* htop, const float* keys,
                              int key_ld, const float* mem, int val_ld, const int* lens, int S_max, int H, int K,
                              int CH, int SC, XOut xo, const int* done, StepCtl ctl, AttFold fo) {
  auto fn = attention_cluster_kernel<KMAX, JPT>;
  cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = dim3(kAttThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  attr[1].id = cudaLaunchAttributeClusterDimension;
  attr[1].val.clusterDim.x = nch;
  attr[1].val.clusterDim.y = 1;
  attr[1].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 2;
  return cudaLaunchKernelEx(&cfg, fn, htop, keys, key_ld, mem, val_ld, lens, S_max, H, K, CH, SC, xo, done, ctl, fo);
}

struct AttPlan {
  int nch, CH, SC;
  size_t smem;
};

// Launch plan: the largest nch (<= att_nch) whose B clusters of nch CTAs are all co-resident
// (cudaOccupancyMaxActiveClusters: clusters must fit inside a GPC, 1 CTA per SM at this shared
// memory size) - a second wave of clusters would double the kernel time.
template <int KMAX, int JPT>
static AttPlan att_plan(int B, int S_max, int H, int K, int key_ld, int val_ld, bool same, int num_sms, AttFold& fo) {
  auto fn = attention_cluster_kernel<KMAX, JPT>;
  const char* forced = std::getenv("ONMT_ATT_NCH");
  AttPlan p{};
  for (int nch = att_nch(B, S_max, num_sms); nch >= 1; --nch) {
    const int CH = (S_max + nch - 1) / nch;
    const int kl = same ? val_ld : key_ld;
    auto r4 = [](size_t n) { return (n + 3) & ~(size_t)3; };
    auto bytes = [&](int SC) {
      return (r4((size_t)K * H) + 3 * 16 + 16 * kSCMax + 2 * (r4((size_t)SC * val_ld) + (same ? 0 : r4((size_t)SC * kl)))) * 4;
    };
    size_t extra = 0;                              // folded W_out: prefetched tile shares
    if (fo.wpart) extra = (size_t)fo.n_wt * K * ((H / 4 + nch - 1) / nch) * 16;
    const size_t esave = fo.att_out ? r4((size_t)K * CH) * 4 : 0;   // attention output: raw scores
    // positions per sub-chunk: the largest of 16 / 12 / 8 that fits (fewer sub-chunks = fewer
    // barriers; c4's H = 1000 rows fit 12)
    const int SC = bytes(16) + extra + esave <= 220 * 1024 ? 16 : bytes(12) + extra + esave <= 220 * 1024 ? 12 : 8;
    // push combine (8 chunks or K >= 8) only when its receive buffer fits next to the rest;
    // otherwise the pull combine (no receive buffer)
    const bool vec = (H & 3) == 0 && (kl & 3) == 0 && (val_ld & 3) == 0;
    size_t rbb = (vec && (nch >= 8 || K >= 8)) ? (size_t)nch * K * 16 * ((H / 4 + nch - 1) / nch) : 0;
    if (bytes(SC) + esave + rbb > 220 * 1024) rbb = 0;
    fo.push = rbb > 0;
    fo.pref = bytes(SC) + extra + esave + rbb <= 220 * 1024;
    fo.hp_floats = fo.pref ? (int)(extra / 4) : 0;
    p = AttPlan{nch, CH, SC, bytes(SC) + (fo.pref ? extra : 0) + esave + rbb};
    if (forced || nch == 1) break;
    if (cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)p.smem) != cudaSuccess) break;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(nch, B);
    cfg.blockDim = dim3(kAttThreads);
    cfg.dynamicSmemBytes = p.smem;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = nch;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    int ncl = 0;
    if (cudaOccupancyMaxActiveClusters(&ncl, fn, &cfg) != cudaSuccess) { cudaGetLastError(); break; }
    if (std::getenv("ONMT_ATT_DEBUG"))
      std::fprintf(stderr, "att_plan B=%d S=%d K=%d nch=%d smem=%zu -> %d co-resident clusters\n", B, S_max, K, nch,
                   p.smem, ncl);
    if (ncl >= B) break;
  }
  return p;
}

cudaError_t launch_attention(const float* htop, const float* keys, int key_ld, const float* mem, int val_ld,
                             const int* lens, int B, int S_max, int H, int K, XOut xo, const int* done, int num_sms,
                             StepCtl ctl, cudaStream_t st, AttFold fo) {
  if (H > 4 * kAttThreads || K > kKMax) return cudaErrorInvalidValue;
  const bool same = keys == mem;
#define ONMT_ATT_J(KM, J)                                                                                          \
  {                                                                                                                \
    const AttPlan p = att_plan<KM, J>(B, S_max, H, K, key_ld, val_ld, same, num_sms, fo);                         \
    return launch_att<KM, J>(dim3(p.nch, B), p.nch, p.smem, st, htop, keys, key_ld, mem, val_ld, lens, S_max, H, K, \
                             p.CH, p.SC, xo, done, ctl, fo);                                                       \
  }
#define ONMT_ATT(KM)                 \
  if (H <= 2 * kAttThreads) ONMT_ATT_J(KM, 2) \
  else ONMT_ATT_J(KM, 4)
  if (K <= 1) ONMT_ATT(1);
  if (K <= 2) ONMT_ATT(2);
  if (K <= 4) ONMT_ATT(4);
  if (K == 5) ONMT_ATT(5);                         // (the paper's beam size: no predicated-off rows)
  if (K <= 8) ONMT_ATT(8);
  if (K == 10) ONMT_ATT(10);                       // (BASELINE c5)
  ONMT_ATT(16);
#undef ONMT_ATT
#undef ONMT_ATT_J
}

}  // namespace onmt
