// model.h — launchers of the decode-step kernels (model.cu, attn.cu, gemm_tc.cu).
#pragma once
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <stdint.h>
#include <algorithm>
#include <limits.h>

namespace rt {
typedef __nv_bfloat16 bf16;

// ---- row / elementwise kernels (model.cu)
void launch_init_weights(bf16* out, int64_t n, uint64_t seed, int32_t tensor_id, float sigma, cudaStream_t s);
// W_gate_up stored with rows interleaved per 128-row tile: [64 gate | 64 up] (EPI_SWIGLU)
void launch_init_weights_gu(bf16* out, int ff, int d, uint64_t seed, int32_t tensor_id, float sigma,
                            cudaStream_t s);
// UMMA-tiled weights: 128 x 64 bf16 tiles (16 KiB, SW128 image), tile (mt, kb) at mt*KB+kb;
// gu_ff > 0 interleaves gate/up rows per tile.  Buffer size ceil(M/128)*128*K elements.
void launch_init_weights_tiled(bf16* out, int M, int K, int gu_ff, uint64_t seed, int32_t tensor_id, float sigma,
                               cudaStream_t s);
void launch_pack_tiled(const bf16* src, bf16* dst, int M, int K, cudaStream_t s);
inline int64_t tiled_elems(int M, int K) { return (int64_t)((M + 127) / 128) * 128 * K; }
void launch_embed_norm(const int32_t* row_tok, int row0, int n, const bf16* emb, int d, float* x, bf16* h,
                       cudaStream_t s);
// h[n] = bf16(x[n] * rsqrt(sum_t ss[n][t] / d + eps)), ss: [n][n_tiles] partial sums of squares
void launch_norm_apply(const float* x, const float* ss, int n_tiles, int n, int d, bf16* h, cudaStream_t s);
void launch_gather_rows(const int32_t* slot_row, int B, int row0, int n, const bf16* h, int d, bf16* hfin,
                        cudaStream_t s);
void launch_argmax_reduce(const float* pv, const int32_t* pi, int n_mtiles, int N, int32_t* tok,
                          cudaStream_t s);
void launch_kv_write(void* pool, const bf16* k, const bf16* v, const int32_t* slot, int n, int nkv, int hd,
                     cudaStream_t s);
void launch_kv_read(const void* pool, bf16* out, int n_pages, int nkv, int hd, cudaStream_t s);

// ---- paged decode attention (attn.cu)
struct AttnArgs {
  const bf16* q;            // [n_rows][nq][hd]  (rows of this launch)
  const void* pool;         // this layer's pool
  const int32_t* page_table;
  int pt_stride;
  const int32_t* row_task;  // indexed by row0 + r
  const int32_t* row_pos;   // seqlen = pos + 1   (when row_seqlen == nullptr)
  const int32_t* row_seqlen;
  int row0, n_rows, nq, nkv, hd, G;
  int chunk_pages, max_chunks;
  bf16* out;                // [n_rows][nq][hd]
  float* out_f32;           // nullable, indexed by global row (row0 + r)
  float* ws;                // split-KV partials [rows][nq][max_chunks][hd + 2]
  int* tickets;             // [rows][nkv] zero-initialised, self-resetting (split-KV merge)
  float scale_log2;
};
int64_t attn_ws_floats(int n_rows, int nq, int hd, int max_chunks);
void attn_plan(int n_rows, int nkv, int max_seqlen, int* chunk_pages, int* max_chunks);
void launch_attention(const AttnArgs& a, cudaStream_t s);

// ---- tcgen05 GEMM with fused epilogues (gemm_tc.cu)
struct TmaMap {
  alignas(64) unsigned char bytes[128];
};
bool make_tma_2d_bf16(TmaMap* out, const void* base, uint64_t inner, uint64_t rows, uint32_t box_inner,
                      uint32_t box_rows);
struct GemmTmaSet {       // activation operand: one map per supported N tile
  TmaMap m32, m64, m128, m256;
  int rows_cap;
};
bool make_gemm_act_maps(GemmTmaSet* out, const void* base, int K, int rows_cap);

enum EpiMode { EPI_STORE = 0, EPI_ARGMAX = 1, EPI_QKV = 2, EPI_RESID = 3, EPI_SWIGLU = 4 };

struct QkvFuse {
  const int32_t *row_task, *row_pos, *page_table;
  int row0, pt_stride, nq, nkv, hd;
  const float *cos, *sin;
  bf16* q_out;     // [n][nq][hd] (rows of this launch)
  void* pool;      // this layer's pool
  float* q_cap;    // nullable, [global row][nq][hd]
};

struct GemmArgs {
  const bf16* w;      // UMMA-tiled weights (launch_init_weights_tiled / launch_pack_tiled)
  int M, N, K, kb_total, m_tiles, mode;
  float* out;         // EPI_STORE [N][M]; EPI_ARGMAX logits [N][M] or null
  float* part_val;    // EPI_ARGMAX [m_tiles][N]
  int32_t* part_idx;
  float* x;           // EPI_RESID residual [N][M]
  float* ss;          // EPI_RESID [N][m_tiles]
  bf16* act;          // EPI_SWIGLU [N][ff]
  int ff;
  QkvFuse qkv;        // EPI_QKV
};
int gemm_bn(int N);
int gemm_choose_splits(int M, int N, int K);   // cluster split-K factor (1..16)
// splits <= 0: gemm_choose_splits
cudaError_t launch_gemm_epi(const bf16* w_tiled, const GemmTmaSet& xmaps, GemmArgs g, int splits, cudaStream_t s);
}  // namespace rt
