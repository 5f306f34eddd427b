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
// first-chunk embedding launched before the plan handshake (row count read on the device)
void launch_embed_plan(const int32_t* row_tok, const int32_t* n_rows_dev, int fwd_rows, const bf16* emb, int d,
                       float* x, bf16* xb, float* ss, cudaStream_t s);
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
  // QKV folded into the decode attention (nullable part): the projection's split-K partials
  // part[s][r][m] (s < part_splits, r < part_ld_n rows, m < part_m = (nq + 2 nkv) hd in the
  // weights' physical row order: within a head rows 2i, 2i + 1 = dims i, i + hd/2), summed in
  // split order, scaled by the row's RMSNorm rsqrt(sum_t rs_ss[r][t] / d_model + 1e-5), RoPE
  // on q and k (cos / sin [pos][hd/2]); bf16 q -> q_out (and fp32 -> q_cap[row0 + r], nullable),
  // bf16 k / v appended into the row's page at its position (the pool above, writable)
  const float* part;
  int part_splits, part_ld_n, part_m;
  const float* rs_ss;
  int rs_tiles, d_model;
  const float *cos, *sin;
  bf16* q_out;
  float* q_cap;
};
int64_t attn_ws_floats(int n_rows, int nq, int hd, int max_chunks);
void attn_plan(int n_rows, int nkv, int max_seqlen, int* chunk_pages, int* max_chunks);
void launch_attention(const AttnArgs& a, cudaStream_t s);
// the folded QKV epilogue (a.part, ...) for the prompt rows of SchedParams::pf_tiles
void launch_qkv_finish(const AttnArgs& a, const int4* tiles, int n_tiles, cudaStream_t s);

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
  int groups;               // warp groups per CTA (0: by load, 1 / 2 forced)
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

enum EpiMode { EPI_STORE = 0, EPI_ARGMAX = 1, EPI_QKV = 2, EPI_RESID = 3, EPI_SWIGLU = 4, EPI_PART = 5 };
// projection kernel paths (GemmArgs::force_path; the values of rt.h RT_GEMM_PATH_*):
// AUTO = measured dispatch; SPLITK = k_gemm_tc (cluster split-K / one tile per CTA);
// STREAMK = k_gemm_sk (hybrid data-parallel + stream-K, N > 128); PAIR = k_gemm_2sm (CTA pairs, N > 128)
// DEC = k_gemm_dec (CTA pairs + cluster split-K, N <= 256, few pair-tiles)
enum GemmPath { GEMM_PATH_AUTO = 0, GEMM_PATH_SPLITK = 1, GEMM_PATH_STREAMK = 2, GEMM_PATH_PAIR = 3, GEMM_PATH_DEC = 4 };

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
  int l2_evict_first;  // set by launch_gemm_epi: weight tiles are read once per step
  // EPI_PART (decode QKV folded into the attention): split s of the cluster / pair
  // split-K writes its raw fp32 partial to part[s][n][m] (rows n < N, ld_n rows per split);
  // the attention kernel sums the splits, applies the RMSNorm scale and RoPE, appends K/V
  float* part;
  int part_ld_n;
  // set by launch_gemm_epi: CTA (x, y) runs linear tile tile0 + y of the GEMM's m_tiles x
  // n_tiles tiles (n fastest: the n-tiles of one m-tile are adjacent and the later ones read
  // the weight tile from L2); tile_count tiles in this launch
  int n_tiles, tile0, tile_count;
  // stream-K workspace for N > 128 rows (nullable: one tile per CTA): partial tiles
  // [SMs][2][256][128] fp32 (gemm_sk_ws_floats) and zeroed self-resetting tile tickets
  float* sk_ws;
  unsigned* sk_cnt;
  int sk_cnt_cap;
  // kernel choice overrides (parity tests / the tuner; 0 = the measured dispatch): the N
  // tile width and the path (GEMM_PATH_*)
  int force_bn, force_path;
  // decode-pair split-K exchange (k_gemm_dec; nullable: the kernel is not used): fp32
  // workspace of gemm_dec_ws_floats(M, N) floats, epoch flags [pair-tiles][2][splits] (zeroed
  // once), and an epoch that the caller increments before every launch
  float* dec_ws;
  int64_t dec_ws_floats;
  unsigned* dec_flags;
  int dec_flags_cap;
  unsigned dec_epoch;
};
// floats of the k_gemm_dec workspace for an [M x K] projection at N rows (0: not used)
int64_t gemm_dec_ws_floats(int M, int N, int K);
constexpr int kDecFlags = 512;  // epoch flags of the k_gemm_dec exchange (pair-tiles x 2 x splits)
int64_t gemm_sk_ws_floats();
int gemm_bn(int M, int K, int N);
int gemm_choose_splits(int M, int N, int K);   // cluster split-K factor (1..16)
int gemm_part_splits(int M, int K, int N);  // EPI_PART partial count (0: unsupported)
// x[n][:] += sum_s part[s][n][:] (split order), xb = bf16(x), ss[n][M/128] sums of squares
void launch_resid_reduce(const float* part, int S, int ld_n, int N, int M, float* x, bf16* xb, float* ss,
                         cudaStream_t s);
// splits <= 0: gemm_choose_splits
cudaError_t launch_gemm_epi(const bf16* w_tiled, const GemmTmaSet& xmaps, GemmArgs g, int splits, cudaStream_t s);

// ---- device trace buffers (common.cuh TraceScope), one binder per translation unit
void trace_bind_model(void* rec, unsigned* n, unsigned cap);
void trace_bind_attn(void* rec, unsigned* n, unsigned cap);
void trace_bind_gemm(void* rec, unsigned* n, unsigned cap);
void trace_bind_sched(void* rec, unsigned* n, unsigned cap);
}  // namespace rt
