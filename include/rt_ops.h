/* rt_ops.h — op-level C ABI of the hot-path kernels (per-op parity tests and
 * microbenchmarks).  Every pointer named d_* is a DEVICE pointer (the caller
 * owns the allocation, e.g. a torch.cuda tensor); `stream` is a cudaStream_t
 * (NULL = legacy default stream).  All calls are asynchronous on `stream` and
 * return rt_status (RT_E_INVAL for bad shapes, RT_E_CUDA on launch failure).
 *
 * KV page layout: one layer's pool is
 *   [n_pages][n_kv_heads][2 (K,V)][16 tokens][head_dim] bf16,
 * each 16 x head_dim block stored with the 16-byte-chunk XOR swizzle
 *   phys_chunk = chunk ^ ((tok >> s) & m)   (hd=128/64: s=0, m=7; hd=32: s=1, m=3)
 * so that one cp.async.bulk of a (page, kv head) lands conflict-free for ldmatrix.
 */
#ifndef RT_OPS_H_
#define RT_OPS_H_
#include <stdint.h>
#include "rt.h"

#ifdef __cplusplus
extern "C" {
#endif

/* a7 paged decode attention (PAPER.md:387 PagedAttention; BASELINE.json
 * "paged-KV ('context cache') attention decode").  For each row r:
 *   o[r, h] = softmax(q[r, h] . K[0:seqlen[r]]^T / sqrt(hd)) V[0:seqlen[r]],
 *   K/V of kv head h / G from pages page_table[row_task[r] * pt_stride + p / 16].
 * d_q bf16 [n_rows][n_q][hd]; d_out bf16 [n_rows][n_q][hd]; d_out_f32 (nullable)
 * fp32 same shape; d_ws workspace >= rt_op_attention_ws_bytes(...), ZERO-FILLED before
 * its first use (it holds self-resetting split-KV merge tickets, left zero on return).
 * hd in {32, 64, 128}; G = n_q / n_kv in {1..8}. */
rt_status rt_op_paged_attention(const void* d_q, const void* d_pool, const int32_t* d_page_table,
                                int32_t pt_stride, const int32_t* d_row_task,
                                const int32_t* d_row_seqlen, int32_t n_rows, int32_t max_seqlen,
                                int32_t n_q, int32_t n_kv, int32_t hd, void* d_out, float* d_out_f32,
                                void* d_ws, int64_t ws_bytes, void* stream);
int64_t rt_op_attention_ws_bytes(int32_t n_rows, int32_t max_seqlen, int32_t n_q, int32_t hd);

/* a5 causal prefill attention over paged KV (NEXT-1; the prompt rows of k = 0 admissions,
 * PAPER.md:72, 93 "Decoding 0" includes the prefill): d_tiles int32 [n_tiles][4] = (first row,
 * rows <= 16, pos0, task): rows first_row .. first_row + rows - 1 are the consecutive positions
 * pos0 .. pos0 + rows - 1 (pos0 a multiple of 16) of task's prompt, each attending causally to
 * positions 0 .. its own (pages from page_table[task * pt_stride + p / 16], which must already
 * hold the K/V of every attended position).  d_q bf16 [n_rows][n_q][hd]; d_out bf16 same shape;
 * d_out_f32 (nullable) fp32 same shape.  groups: warp groups per CTA (0: by load, 1 or 2).
 * hd in {32, 64, 128}; G = n_q / n_kv in {1..8}. */
rt_status rt_op_prefill_attention(const void* d_q, const void* d_pool, const int32_t* d_page_table,
                                  int32_t pt_stride, const int32_t* d_tiles, int32_t n_tiles, int32_t n_rows,
                                  int32_t n_q, int32_t n_kv, int32_t hd, int32_t groups, void* d_out,
                                  float* d_out_f32, void* stream);

/* Write logical K/V rows into the swizzled pool: row r of d_k / d_v (bf16
 * [n_rows][n_kv][hd]) goes to token slot d_slot[r] = page * 16 + offset. */
rt_status rt_op_kv_write(void* d_pool, const void* d_k, const void* d_v, const int32_t* d_slot,
                         int32_t n_rows, int32_t n_kv, int32_t hd, void* stream);
/* Inverse: read logical [n_pages][2][n_kv][16][hd] bf16 out of the swizzled pool. */
rt_status rt_op_kv_read(const void* d_pool, void* d_out, int32_t n_pages, int32_t n_kv, int32_t hd,
                        void* stream);

/* KV eviction / restore copies (PAPER.md:226-229 context caching; DESIGN.md R-EVICT):
 * d_swap int32 [n][4] = (dir 0 device->host / 1 host->device, task (unused), device page,
 * host page); for every layer l < n_layers the (page, layer) block of blk_bytes =
 * n_kv * 2 * 16 * hd * 2 bytes is copied between layer l of the device pool (layer stride
 * pool_layer_bytes) and host page h at h_host + (h * n_layers + l) * blk_bytes.  h_host is a
 * page-locked host allocation addressable from the device (cudaHostAlloc / pinned memory under
 * UVA): the copy is zero-copy over PCIe.  Entries of one call must not read a page another
 * entry of the same call writes. */
rt_status rt_op_kv_swap(const int32_t* d_swap, int32_t n, void* d_pool, int64_t pool_layer_bytes, void* h_host,
                        int64_t blk_bytes, int32_t n_layers, void* stream);

/* a6 dense projection on tcgen05 (UMMA 128 x BN x 16, TMEM accumulator, TMA SW128):
 *   d_out[n][m] = sum_k W[m, k] * X[n, k]     fp32; split-K over a cluster of
 *   `splits` CTAs per tile (1..16, <= K/64), reduced through distributed shared
 *   memory in rank order (deterministic); splits <= 0 picks the engine's choice.
 * d_w bf16 [M][K] row-major, d_x bf16 [N][K] row-major (n_cap >= N rows allocated),
 * K % 64 == 0. */
rt_status rt_op_gemm(const void* d_w, const void* d_x, float* d_out, int32_t M, int32_t N, int32_t K,
                     int32_t n_cap, int32_t splits, void* stream);

/* The engine's weight layout: pack a row-major bf16 [M][K] matrix into
 * UMMA-ready 128 x 64 tiles (d_dst holds ceil(M/128)*128*K elements), and run the
 * projection directly on a packed matrix (same semantics as rt_op_gemm).  path = RT_GEMM_PATH_*
 * (AUTO: the engine's dispatch; a forced path falls back to SPLITK where it does not apply),
 * bn = N tile width (0: by the dispatch; 32 / 64 / 128 / 160 / 192 / 256). */
rt_status rt_op_pack_tiled(const void* d_src, void* d_dst, int32_t M, int32_t K, void* stream);
rt_status rt_op_gemm_tiled(const void* d_w_tiled, const void* d_x, float* d_out, int32_t M, int32_t N,
                           int32_t K, int32_t n_cap, int32_t splits, int32_t path, int32_t bn, void* stream);

/* a8 lm_head + greedy argmax (lowest index on ties) over the vocabulary:
 * d_tok[n] = argmax_m sum_k W[m,k] X[n,k]; d_logits (nullable) fp32 [N][M]. */
rt_status rt_op_lm_argmax(const void* d_w, const void* d_x, int32_t M, int32_t N, int32_t K,
                          int32_t n_cap, int32_t* d_tok, float* d_logits, void* d_ws,
                          int64_t ws_bytes, void* stream);

/* Counter-based init (DESIGN.md AMB-15): d_out bf16 [n] holds the weights of
 * tensor_id at flat indices [0, n). */
rt_status rt_op_init_weights(void* d_out, int64_t n, uint64_t seed, int32_t tensor_id, float sigma,
                             void* stream);

/* a2 Eq. 4 priority for n tasks (fp64, fixed op order). */
rt_status rt_op_priority(const int64_t* d_t_ref_d_ert /* [n][4]: t, ref, D, ERT */,
                         const int32_t* d_k, const double* d_alpha, const double* d_beta, int32_t n,
                         int32_t g_us, int32_t net_us, int32_t eps_l_us, double* d_pri, void* stream);

/* a12 global ordering across replicas (BASELINE.json "one NCCL allgather ... per scheduling
 * round so the global utility ordering stays exact"; DESIGN.md AMB-22): the device merge the
 * engine runs on the allgathered candidates.  d_all fp64 [world][16][4] = per-rank top-16
 * candidate records (pri, arrival_us, global request id, rank), rid < 0 = empty slot;
 * d_merged fp64 [16][4] receives the top 16 of the union by (pri desc, arrival asc, rid asc),
 * empty slots last.  1 <= world <= 8. */
rt_status rt_op_merge_candidates(const double* d_all, int32_t world, double* d_merged, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* RT_OPS_H_ */
