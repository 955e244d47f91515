// Split-K tcgen05 GEMM with the split reduction done inside a thread-block cluster and the
// consumer fused in (decoder LSTM cell, PAPER.md P129-136; or h~ = tanh(W_out [c; h]),
// P69).  Cluster = the S split-K CTAs of one 128-row weight tile: each CTA streams its
// K-slice (TMA -> smem -> tcgen05.mma, hi/lo activation planes into one fp32 TMEM
// accumulator), parks its partial tile in its own shared memory, and after a cluster
// barrier CTA s reduces rows [s*128/S, (s+1)*128/S) over all S partials through
// distributed shared memory in fixed order (deterministic), then applies the epilogue.
// Removes the separate cell / tanh launches and the partial round trip through L2.
#include "common.cuh"
#include "ptx.cuh"

namespace onmt {

enum { EPI_CELL = 0, EPI_TANH = 1 };

struct FusedArgs {
  int n_rows_pad, n_group, n_valid, k_blocks, kb_per_split, stages, tmem_cols, S;
  int M;                   // valid weight rows (4H for the cell, H for tanh)
  // EPI_CELL
  const float4* bias;      // [H] interleaved (i,f,g,o) pre-summed biases
  const float* cg;         // [rows_pad][H] c_prev gathered by parent
  float* c_out;
  float* h_out;
  int H;
  CellDst dst;
  // EPI_TANH
  float* htilde;
  XOut xg;
  StepCtl ctl;
};

__device__ __forceinline__ float4 ld_peer_f4(const float* local, uint32_t peer) {
  uint32_t ra;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(smem_u32(local)), "r"(peer));
  float4 v;
  asm volatile("ld.shared::cluster.v4.f32 {%0, %1, %2, %3}, [%4];"   // ordered after the cluster barrier
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)                // (volatile), independent otherwise
               : "r"(ra));
  return v;
}

// sigmoid / tanh via the fast exponential (ex2.approx, rel. error ~2^-21): well inside the
// fp32 (1e-5) and bf16 (2e-3) log-prob bars; avoids the IEEE-division / tanhf slow paths
__device__ __forceinline__ float sigmf(float x) { return __frcp_rn(1.f + __expf(-x)); }
__device__ __forceinline__ float tanhfast(float x) {
  const float e = __expf(-2.f * fabsf(x));
  const float t = (1.f - e) * __frcp_rn(1.f + e);
  return copysignf(t, x);
}

template <int EPI>
__global__ void __launch_bounds__(128, 1)
tc_gemm_cluster_kernel(const __grid_constant__ CUtensorMap tmW, const __grid_constant__ CUtensorMap tmX,
                       FusedArgs a) {
  pdl_trigger();
  extern __shared__ __align__(16) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  const uint32_t a_bytes = kTileM * 128, b_bytes = a.n_group * 128;
  const uint32_t stage_bytes = a_bytes + 2 * b_bytes;
  const size_t ring = (size_t)a.stages * stage_bytes;
  const size_t part_bytes = (size_t)a.n_group * kTileM * 4;
  float* part = reinterpret_cast<float*>(smem);                         // [n_group][128] (reuses the ring)
  const int RM = kTileM / a.S;                                          // rows this CTA reduces
  float* red = reinterpret_cast<float*>(smem + (ring > part_bytes ? ring : part_bytes));   // [n_group][RM]
  uint64_t* full = reinterpret_cast<uint64_t*>(red + (size_t)a.n_group * RM);
  uint64_t* empty = full + a.stages;
  uint64_t* done = empty + a.stages;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(done + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t split = cluster_ctarank();
  const int mt = blockIdx.x / a.S;
  const int m0 = mt * kTileM;
  const int n0 = blockIdx.y * a.n_group;
  const int kb0 = split * a.kb_per_split;
  int nkb = a.k_blocks - kb0;
  if (nkb > a.kb_per_split) nkb = a.kb_per_split;
  if (nkb < 0) nkb = 0;

  if (threadIdx.x == 0) {
    tma_prefetch_desc(&tmW);
    tma_prefetch_desc(&tmX);
    for (int s = 0; s < a.stages; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    mbar_init(done, 1);
    fence_mbar_init();
  }
  if (warp == 0) tmem_alloc_dyn(tslot, a.tmem_cols);
  tc_fence_before();
  pdl_wait();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tslot;
  if (all_done(a.ctl)) {
    __syncthreads();
    if (warp == 0) tmem_dealloc(tmem, a.tmem_cols);
    return;
  }

  if (warp == 0 && lane == 0) {
    for (int i = 0; i < nkb; ++i) {
      const int s = i % a.stages;
      if (i >= a.stages) mbar_wait(&empty[s], ((i / a.stages) & 1) ^ 1);
      uint8_t* st = smem + s * stage_bytes;
      mbar_arrive_expect_tx(&full[s], stage_bytes);
      const int kx = (kb0 + i) * kBK;
      tma_load_2d(st, &tmW, kx, m0, &full[s]);
      tma_load_2d(st + a_bytes, &tmX, kx, n0, &full[s]);
      tma_load_2d(st + a_bytes + b_bytes, &tmX, kx, a.n_rows_pad + n0, &full[s]);
    }
  } else if (warp == 1 && lane == 0) {
    const uint32_t idesc = umma_idesc_bf16(kTileM, a.n_group);
    for (int i = 0; i < nkb; ++i) {
      const int s = i % a.stages;
      mbar_wait(&full[s], (i / a.stages) & 1);
      tc_fence_after();
      const uint32_t sa = smem_u32(smem + s * stage_bytes);
      const uint32_t sbh = sa + a_bytes, sbl = sa + a_bytes + b_bytes;
#pragma unroll
      for (int kk = 0; kk < kBK / 16; ++kk) {
        const uint64_t da = umma_desc_sw128(sa + kk * 32);
        tc_mma_bf16(tmem, da, umma_desc_sw128(sbh + kk * 32), idesc, (i | kk) != 0);
        tc_mma_bf16(tmem, da, umma_desc_sw128(sbl + kk * 32), idesc, 1u);
      }
      tc_commit(&empty[s]);
    }
    tc_commit(done);
  }
  __syncwarp();
  if (nkb > 0) {
    mbar_wait(done, 0);
    tc_fence_after();
  }
  __syncthreads();                               // ring no longer read by the tensor core
  // ---- park the partial tile: part[n][m] (column-major over TMEM lanes: conflict-free)
  {
    const int q = warp & 3;
    const uint32_t trow = tmem + ((uint32_t)(q * 32) << 16);
    const int m = q * 32 + lane;
    for (int c0 = 0; c0 < a.n_group; c0 += 16) {
      float v[16];
      if (nkb > 0) {
        tmem_ld16(trow + c0, v);
      } else {
#pragma unroll
        for (int j = 0; j < 16; ++j) v[j] = 0.f;
      }
#pragma unroll
      for (int j = 0; j < 16; ++j) part[(c0 + j) * kTileM + m] = v[j];
    }
  }
  tc_fence_before();
  cluster_sync_all();
  // ---- reduce my RM rows over the S partials (fixed peer order) into red[n][RM]
  const int mr0 = split * RM;
  const int RM4 = RM / 4;
  for (int it0 = threadIdx.x; it0 < a.n_group * RM4; it0 += 2 * blockDim.x) {
    float4 v[2][8];                               // 2 items x 8 peers of remote loads in flight
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const int it = min(it0 + u * (int)blockDim.x, a.n_group * RM4 - 1);
      const int n = it / RM4, m4 = (it % RM4) * 4;
      const float* loc = part + n * kTileM + mr0 + m4;
#pragma unroll
      for (int p = 0; p < 8; ++p) v[u][p] = p < a.S ? ld_peer_f4(loc, p) : make_float4(0.f, 0.f, 0.f, 0.f);
    }
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const int it = it0 + u * blockDim.x;
      if (it >= a.n_group * RM4) break;
      const int n = it / RM4, m4 = (it % RM4) * 4;
      float4 acc = v[u][0];                       // fixed peer order: deterministic
#pragma unroll
      for (int p = 1; p < 8; ++p) { acc.x += v[u][p].x; acc.y += v[u][p].y; acc.z += v[u][p].z; acc.w += v[u][p].w; }
      *reinterpret_cast<float4*>(red + n * RM + m4) = acc;
    }
  }
  __syncthreads();
  // ---- fused epilogue on rows [m0 + mr0, m0 + mr0 + RM)
  if (EPI == EPI_CELL) {
    const int U = RM / 4;                        // LSTM units in my rows (rows 4u+g interleaved)
    const int u0 = (m0 + mr0) / 4;
    const int nit = U * a.n_group;
    for (int b0 = threadIdx.x; b0 < nit; b0 += 4 * blockDim.x) {
      float4 bb[4];
      float cp[4];
#pragma unroll
      for (int v = 0; v < 4; ++v) {               // all global loads of 4 items first
        const int it = b0 + v * blockDim.x;
        const int ul = it % U, n = it / U;
        const int r = n0 + n, j = u0 + ul;
        const bool ok = it < nit && r < a.n_valid && j < a.H;
        bb[v] = ok ? __ldg(&a.bias[j]) : make_float4(0.f, 0.f, 0.f, 0.f);
        cp[v] = ok ? __ldg(&a.cg[(size_t)r * a.H + j]) : 0.f;
      }
#pragma unroll
      for (int v = 0; v < 4; ++v) {
        const int it = b0 + v * blockDim.x;
        const int ul = it % U, n = it / U;
        const int r = n0 + n, j = u0 + ul;
        if (!(it < nit && r < a.n_valid && j < a.H)) continue;
        const float* gz = red + n * RM + 4 * ul;
        const float i_ = sigmf(gz[0] + bb[v].x), f_ = sigmf(gz[1] + bb[v].y), g_ = tanhfast(gz[2] + bb[v].z),
                    o_ = sigmf(gz[3] + bb[v].w);
        const float c = f_ * cp[v] + i_ * g_;
        const float h = o_ * tanhfast(c);
        a.c_out[(size_t)r * a.H + j] = c;
        a.h_out[(size_t)r * a.H + j] = h;
        for (int d = 0; d < a.dst.n; ++d) store_x(a.dst.x[d], r, a.dst.col[d] + j, h);
      }
    }
  } else {
    for (int it = threadIdx.x; it < RM * a.n_group; it += blockDim.x) {
      const int ml = it % RM, n = it / RM;
      const int r = n0 + n, j = m0 + mr0 + ml;
      if (r >= a.n_valid || j >= a.M) continue;
      const float h = tanhfast(red[n * RM + ml]);
      a.htilde[(size_t)r * a.M + j] = h;
      store_x(a.xg, r, j, h);
    }
  }
  cluster_sync_all();                            // peers finished reading my partial
  if (warp == 0) tmem_dealloc(tmem, a.tmem_cols);
}

static size_t fused_smem_bytes(int n_group, int stages, int S) {
  const size_t ring = (size_t)stages * (kTileM * 128 + 2 * (size_t)n_group * 128);
  const size_t part = (size_t)n_group * kTileM * 4;
  return 1024 + (ring > part ? ring : part) + (size_t)n_group * (kTileM / S) * 4 + (2 * stages + 1) * 8 + 16;
}

template <int EPI>
static cudaError_t launch_fused(const CUtensorMap& tmW, const CUtensorMap& tmX, const FusedArgs& a, int m_tiles,
                                int n_groups, cudaStream_t st) {
  const size_t smem = fused_smem_bytes(a.n_group, a.stages, a.S);
  auto fn = tc_gemm_cluster_kernel<EPI>;
  cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(m_tiles * a.S, n_groups);
  cfg.blockDim = dim3(128);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  attr[1].id = cudaLaunchAttributeClusterDimension;
  attr[1].val.clusterDim.x = a.S;
  attr[1].val.clusterDim.y = 1;
  attr[1].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 2;
  return cudaLaunchKernelEx(&cfg, fn, tmW, tmX, a);
}

template <int EPI>
static int max_active_clusters(int n_group, int stages, int S) {
  static int cache[2][9][512 / 16 + 1][5] = {};
  int& c = cache[EPI][S][n_group / 16][stages];
  if (c) return c;
  const size_t smem = fused_smem_bytes(n_group, stages, S);
  auto fn = tc_gemm_cluster_kernel<EPI>;
  cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(S * 64);
  cfg.blockDim = dim3(128);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = S;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  int n = 0;
  if (cudaOccupancyMaxActiveClusters(&n, fn, &cfg) != cudaSuccess || n < 1) n = 1;
  c = n;
  return n;
}

template <int EPI>
static void fill_common(FusedArgs& a, int n_rows_pad, int n_group, int n_valid, int k_blocks, int M, int m_tiles) {
  a.n_rows_pad = n_rows_pad;
  a.n_group = n_group;
  a.n_valid = n_valid;
  a.k_blocks = k_blocks;
  const int groups = n_rows_pad / n_group;
  int S = 8;
  for (;; S >>= 1) {
    if (S == 1) break;
    if ((k_blocks + S - 1) / S * (S - 1) >= k_blocks) continue;            // every split gets >= 1 block
    const int kbps = (k_blocks + S - 1) / S;
    int st = kbps < 4 ? kbps : 4;
    while (st > 1 && fused_smem_bytes(n_group, st, S) > 227 * 1024) --st;
    if (m_tiles * groups <= max_active_clusters<EPI>(n_group, st, S)) break;   // one wave of clusters
  }
  a.S = S;
  a.kb_per_split = (k_blocks + S - 1) / S;
  int stages = a.kb_per_split < 4 ? a.kb_per_split : 4;
  while (stages > 1 && fused_smem_bytes(n_group, stages, S) > 227 * 1024) --stages;
  a.stages = stages < 1 ? 1 : stages;
  int tc = 32;
  while (tc < n_group) tc <<= 1;
  a.tmem_cols = tc;
  a.M = M;
}

// decoder LSTM layer: gates = W [x; h] (+ bias), cell update, h written to dst operands
cudaError_t tc_gemm_cell(const CUtensorMap& tmW, const CUtensorMap& tmX, int m_pad, int n_rows_pad, int n_group,
                         int n_valid, int k_blocks, const float* bias, const float* cg, float* c_out, float* h_out,
                         int H, CellDst dst, StepCtl ctl, cudaStream_t st) {
  FusedArgs a{};
  fill_common<EPI_CELL>(a, n_rows_pad, n_group, n_valid, k_blocks, 4 * H, m_pad / kTileM);
  a.bias = reinterpret_cast<const float4*>(bias);
  a.cg = cg;
  a.c_out = c_out;
  a.h_out = h_out;
  a.H = H;
  a.dst = dst;
  a.ctl = ctl;
  return launch_fused<EPI_CELL>(tmW, tmX, a, m_pad / kTileM, n_rows_pad / n_group, st);
}

// attentional vector: h~ = tanh(W_out [c; h])
cudaError_t tc_gemm_tanh(const CUtensorMap& tmW, const CUtensorMap& tmX, int m_pad, int n_rows_pad, int n_group,
                         int n_valid, int k_blocks, int H, float* htilde, XOut xg, StepCtl ctl, cudaStream_t st) {
  FusedArgs a{};
  fill_common<EPI_TANH>(a, n_rows_pad, n_group, n_valid, k_blocks, H, m_pad / kTileM);
  a.htilde = htilde;
  a.xg = xg;
  a.ctl = ctl;
  return launch_fused<EPI_TANH>(tmW, tmX, a, m_pad / kTileM, n_rows_pad / n_group, st);
}

}  // namespace onmt
