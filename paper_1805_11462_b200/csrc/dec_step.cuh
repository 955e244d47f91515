// Host/device interface of the fused decoder-step kernel (dec_step.cu).
#pragma once
#include "common.cuh"

namespace onmt {

constexpr int kDsMaxGemm = 5;       // up to 4 decoder layers + W_out
constexpr int kDsMaxKbps = 4;       // K blocks per split (weight slots of a phase)
constexpr int kDsBarsPerPhase = 3 + kDsMaxKbps;   // wbar, full[kbps], done, rbar

struct DsGemm {
  CUtensorMap tmW, tmX;
  int S, NC, kbps, k_blocks, tiles, n_group, n_rows_pad, n_valid, M;
  uint32_t w_off;                   // shared offset of the weight slots (kbps x 16 KB)
  float* scratch;                   // [tiles][S][n_group][128] partial tiles
  unsigned int* counters;           // [tiles][2] (cta_group_barrier words)
  int epi;                          // 0: LSTM cell, 1: tanh
  const float4* bias;               // cell: [H] interleaved (i, f, g, o)
  const float* cg;                  // cell: gathered c_prev [rows_pad][H]
  float* c_out;
  float* h_out;
  int H;
  CellDst dst;
  float* htilde;                    // tanh: h~ [rows][M] and the generator operand
  XOut xg;
};

struct DsAtt {
  const float* htop;                // [rows][H] (top decoder layer)
  const float* keys;                // 'general': W_in^T m_s [B*S_max][key_ld]; 'dot': == mem
  int key_ld;
  const float* mem;                 // [B*S_max][H]
  const int* lens;
  int B, S_max, H, K, nch, CH, SC;
  XOut xo;                          // W_out operand, context -> columns [0, H)
  const int* done;
  float* part;                      // [B][nch][K][2 + H]: (m, l, ctx) per chunk
};

struct DsArgs {
  DsGemm g[kDsMaxGemm];
  int n_cell;                       // L (phases 0..L-1 are cells, phase L is W_out)
  DsAtt att;
  uint32_t b_off;                   // activation ring / partial receive / attention staging
  uint32_t side_off;                // cell bias + c_prev staging
  uint32_t bar_off;
  unsigned int* gbar;               // grid barrier word
  StepCtl ctl;
};


struct DsGemmSpec {
  const CUtensorMap* tmW;
  const CUtensorMap* tmX;
  int m_pad, n_rows_pad, n_group, n_valid, k_blocks, M;
  float* scratch;
  unsigned int* counters;
  int epi;
  const float* bias;
  const float* cg;
  float* c_out;
  float* h_out;
  int H;
  CellDst dst;
  float* htilde;
  XOut xg;
};

// Plans and (st != nullptr) launches the fused decoder step (cells, attention, W_out);
// cudaErrorInvalidConfiguration when the shapes do not fit.  scratch_floats (optional) is
// raised to the partial-tile scratch the plan needs.
cudaError_t dec_step(const DsGemmSpec* specs, int n_cell, const DsAtt& att, unsigned int* gbar, StepCtl ctl,
                     int num_sms, size_t* scratch_floats, cudaStream_t st);
int dec_step_att_chunks(int B, int S_max, int num_sms);
void dec_step_set_trace(unsigned long long* p);   // (ONMT_KTRACE builds: per-CTA phase stamps)

}  // namespace onmt
