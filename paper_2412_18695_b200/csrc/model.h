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
// UMMA-tiled weights: 128 x 64 bf16 tiles (16 KiB, SW128 image), tile (mt, kb) at mt*KB+kb;
// gu_ff > 0 pairs gate/up rows (row 2k gate, 2k+1 up of feature 64 t + k in tile t);
// rope_hd > 0 pairs the rotate-half partners inside each head (row 2k dim k, 2k+1 dim
// k + hd/2).  Buffer size ceil(M/128)*128*K elements.
void launch_init_weights_tiled(bf16* out, int M, int K, int gu_ff, int rope_hd, uint64_t seed, int32_t tensor_id,
                               float sigma, cudaStream_t s);
void launch_pack_tiled(const bf16* src, bf16* dst, int M, int K, cudaStream_t s);
inline int64_t tiled_elems(int M, int K) { return (int64_t)((M + 127) / 128) * 128 * K; }
// x = emb[tok] (fp32), xb = bf16(x), ss [n][ceil(d/128)] per-tile sums of squares of x
void launch_embed(const int32_t* row_tok, int row0, int n, const bf16* emb, int d, float* x, bf16* xb, float* ss,
                  cudaStream_t s);
// hfin[s] = bf16(RMSNorm(x[slot_row[s] - row0])) from x fp32 and its ss partials
void launch_gather_norm(const int32_t* slot_row, int B, int row0, int n, const float* x, const float* ss, int d,
                        bf16* hfin, cudaStream_t s);
void launch_argmax_reduce(const float* pv, const int32_t* pi, int n_mtiles, int N, int32_t* tok,
                          cudaStream_t s);
void launch_kv_write(void* pool, const bf16* k, const bf16* v, const int32_t* slot, int n, int nkv, int hd,
                     cudaStream_t s);
void launch_kv_read(const void* pool, bf16* out, int n_pages, int nkv, int hd, cudaStream_t s);
// KV eviction / restore copies (swap[i] = (dir 0 to host / 1 to device, task, device page,
// host page)); blk = bytes of one (page, layer) block; host pool [host page][L][blk]
void launch_kv_swap(const int4* swap, int n, void* pool, int64_t pool_layer_bytes, void* host, int64_t blk, int L,
                    cudaStream_t s);

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
  const int32_t* row_list;   // nullable: CTA z serves row row_list[z] (global row; rows
                             // outside [row0, row0 + chunk_rows) are skipped); n_rows = list size
  int chunk_rows;
  int l2_evict_first;        // set by launch_attention: K/V pages are read once per step
};
int64_t attn_ws_floats(int n_rows, int nq, int hd, int max_chunks);
void attn_plan(int n_rows, int nkv, int max_seqlen, int* chunk_pages, int* max_chunks);
void launch_attention(const AttnArgs& a, cudaStream_t s);

// ---- causal prefill attention over paged KV (attn.cu): prompt rows of k = 0 admissions,
// tiles of <= 16 consecutive positions; CTA = (tile, kv head), one warp per q head of the
// GQA group, K/V page blocks shared by the warps through a TMA-fed ring
struct PrefillArgs {
  const bf16* q;            // [n_rows][nq][hd] rows of this forward chunk
  const void* pool;         // this layer's pool
  const int32_t* page_table;
  int pt_stride;
  const int4* tiles;        // (first row, rows, first position, task)
  int n_tiles;
  int row0, n_rows;         // forward chunk: rows outside it are skipped
  int nq, nkv, hd, G;
  bf16* out;                // [n_rows][nq][hd]
  float* out_f32;           // nullable, indexed by global row
  float scale_log2;
  // split-KV (set by launch_attention_prefill from the fields below): CTA (tile, head, chunk)
  // streams chunk `chunk` of the tile's pages; partials -> ws, the last chunk's CTA merges
  int chunks;
  int max_seqlen;           // longest attended context of the launch (chunk plan)
  float* ws;                // nullable: [tiles][nkv][chunks][G][16][hd + 2] fp32
  int64_t ws_floats;
  int* tickets;             // [tiles][nkv] zeroed, self-resetting
  int rotate;               // set by launch_attention_prefill: per-CTA page-walk start
};
void launch_attention_prefill(const PrefillArgs& a, cudaStream_t s);

// ---- tcgen05 GEMM with fused epilogues (gemm_tc.cu)
struct TmaMap {
  alignas(64) unsigned char bytes[128];
};
bool make_tma_2d_bf16(TmaMap* out, const void* base, uint64_t inner, uint64_t rows, uint32_t box_inner,
                      uint32_t box_rows);
struct GemmTmaSet {       // activation operand: one map per supported N tile
  TmaMap m32, m64, m80, m96, m128, m160, m192, m256;  // m80 / m96 / m128: CTA-pair halves
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
  float* ss;          // EPI_RESID [N][m_tiles] per-tile sums of squares of the new x
  bf16* xb;           // EPI_RESID nullable: bf16(new x) [N][M], the next GEMM's operand
  // RMSNorm folded into the epilogue (all modes, nullable): D[m][n] *= rsqrt(sum_t
  // rs_ss[n][t] / K + 1e-5) — the GEMM ran on bf16(x) and the row scale is linear
  const float* rs_ss;
  int rs_tiles;
  bf16* act;          // EPI_SWIGLU [N][ff]
  int ff;
  QkvFuse qkv;        // EPI_QKV
  // L2 prefetch of the NEXT projection's weights (nullable): when its loads are issued,
  // the producer prefetches the first pf_kb k-blocks of every CTA of the next launch
  // (grid pf_S x pf_m_tiles, K = pf_kb_total k-blocks) so that kernel starts on L2 hits
  // while this one drains its pipeline and runs its epilogue (HBM would idle).
  const bf16* pf_w;
  int pf_S, pf_m_tiles, pf_kb_total, pf_kb;
  int l2_evict_first;  // set by launch_gemm_epi: weight tiles are read once per step
  // set by launch_gemm_epi: CTA (x, y) runs linear tile tile0 + y of the GEMM's m_tiles x
  // n_tiles tiles (n fastest: the n-tiles of one m-tile are adjacent and the later ones read
  // the weight tile from L2); tile_count tiles in this launch
  int n_tiles, tile0, tile_count;
  // stream-K workspace for N > 128 rows (nullable: one tile per CTA): partial tiles
  // [SMs][2][256][128] fp32 (gemm_sk_ws_floats) and zeroed self-resetting tile tickets
  float* sk_ws;
  unsigned* sk_cnt;
  int sk_cnt_cap;
};
int64_t gemm_sk_ws_floats();
// fill g.pf_* for a next launch of weights w [M x K] at N columns (splits <= 0: auto),
// prefetching at most budget_bytes in total
void gemm_set_prefetch(GemmArgs& g, const bf16* w, int M, int N, int K, int splits, int64_t budget_bytes);
int gemm_bn(int M, int K, int N);
int gemm_choose_splits(int M, int N, int K);   // cluster split-K factor (1..16)
// splits <= 0: gemm_choose_splits
cudaError_t launch_gemm_epi(const bf16* w_tiled, const GemmTmaSet& xmaps, GemmArgs g, int splits, cudaStream_t s);

// ---- persistent projection chain (gemm_tc.cu): up to 4 dependent decode
// projections (O + residual, gate/up + SwiGLU, down + residual, next layer's QKV + RoPE +
// KV append) in ONE launch of one CTA per SM.  Every job's k-block iterations (m-tile x
// k-block, N <= 64 rows in one 64-wide tile) are split evenly over the CTAs (stream-K);
// weight tiles stream ahead across job boundaries (they do not depend on activations),
// only the activation (X) loads of job j wait for job j - 1 to finish.  Partial tiles
// go to a global workspace; the last contributor of a tile sums them in fixed order and
// runs the fused epilogue.
constexpr int kChainMaxJobs = 4;
struct ChainArgs {
  GemmArgs job[kChainMaxJobs];   // as launch_gemm_epi (w, M, N <= 64, K, mode, epilogue fields)
  TmaMap xmap[kChainMaxJobs];    // activation operand of each job (box 64 x 64)
  float* ws[kChainMaxJobs];      // partial tiles [m_tiles][ws_slots][64][128] fp32
  int ws_slots[kChainMaxJobs];
  unsigned* tile_cnt[kChainMaxJobs];  // [m_tiles] zero-initialised, self-resetting
  unsigned* done;                // [kChainMaxJobs] cumulative finished tiles (never reset)
  unsigned done_target[kChainMaxJobs];  // done[j] value when job j of THIS launch is complete
  int n_jobs;
  int grid;                      // CTAs: <= SM count and <= every job's k-block iterations
  int pf_ahead;                  // weight k-blocks prefetched into L2 beyond the smem ring
};
// max contributors of one m-tile of an (M, K) job over `ctas` CTAs (the ws_slots to allocate)
int chain_slots(int M, int K, int ctas);
// CTAs of a chain over jobs (M[j], K[j]): min(SM count, every job's m-tile x k-block count)
int chain_grid(const int* M, const int* K, int n_jobs);
cudaError_t launch_chain(ChainArgs& a, cudaStream_t s);

// ---- device trace buffers (common.cuh TraceScope), one binder per translation unit
void trace_bind_model(void* rec, unsigned* n, unsigned cap);
void trace_bind_attn(void* rec, unsigned* n, unsigned cap);
void trace_bind_gemm(void* rec, unsigned* n, unsigned cap);
void trace_bind_sched(void* rec, unsigned* n, unsigned cap);
}  // namespace rt
