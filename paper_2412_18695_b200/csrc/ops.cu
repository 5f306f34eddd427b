// ops.cu — op-level C ABI (include/rt_ops.h): the hot-path kernels on caller-owned
// device buffers, for per-op parity tests and microbenchmarks.
#include <mutex>
#include <cuda_runtime.h>
#include <math.h>
#include <stdlib.h>
#include <algorithm>
#include "rt_ops.h"
#include "internal.h"
#include "model.h"

using namespace rt;

namespace rt {
void launch_priority_batch(const int64_t* trde, const int32_t* k, const double* alpha, const double* beta, int n,
                           int g_us, int net_us, int eps_l_us, double* pri, cudaStream_t s);
}

static rt_status last_launch() { return cudaGetLastError() == cudaSuccess ? RT_OK : RT_E_CUDA; }

extern "C" int64_t rt_op_attention_ws_bytes(int32_t n_rows, int32_t max_seqlen, int32_t n_q, int32_t hd) {
  int cp = 0, mc = 0;
  attn_plan(n_rows, 1, max_seqlen, &cp, &mc);
  int mc8 = 0;
  attn_plan(n_rows, 8, max_seqlen, &cp, &mc8);
  mc = mc > mc8 ? mc : mc8;
  const int64_t tk_bytes = (((int64_t)n_rows * n_q * 4) + 255) & ~(int64_t)255;
  return tk_bytes + attn_ws_floats(n_rows, n_q, hd, mc > 8 ? mc : 8) * 4;
}

extern "C" rt_status rt_op_paged_attention(const void* d_q, const void* d_pool, const int32_t* d_page_table,
                                           int32_t pt_stride, const int32_t* d_row_task,
                                           const int32_t* d_row_seqlen, int32_t n_rows, int32_t max_seqlen,
                                           int32_t n_q, int32_t n_kv, int32_t hd, void* d_out, float* d_out_f32,
                                           void* d_ws, int64_t ws_bytes, void* stream) {
  if (n_rows < 0 || max_seqlen < 1 || n_kv < 1 || n_q % n_kv || n_q / n_kv > 8) return RT_E_INVAL;
  if (hd != 32 && hd != 64 && hd != 128) return RT_E_INVAL;
  if (n_rows == 0) return RT_OK;
  AttnArgs a{};
  a.q = (const bf16*)d_q;
  a.pool = d_pool;
  a.page_table = d_page_table;
  a.pt_stride = pt_stride;
  a.row_task = d_row_task;
  a.row_pos = nullptr;
  a.row_seqlen = d_row_seqlen;
  a.row0 = 0;
  a.n_rows = n_rows;
  a.nq = n_q;
  a.nkv = n_kv;
  a.hd = hd;
  a.G = n_q / n_kv;
  attn_plan(n_rows, n_kv, max_seqlen, &a.chunk_pages, &a.max_chunks);
  if (a.max_chunks > 1 && attn_ws_floats(n_rows, n_q, hd, a.max_chunks) * 4 > ws_bytes) {
    a.chunk_pages = (max_seqlen + 15) / 16;
    a.max_chunks = 1;
  }
  a.out = (bf16*)d_out;
  a.out_f32 = d_out_f32;
  // workspace = [merge tickets: n_rows * n_q ints, 256-B padded][split-KV partials]
  const size_t tk_bytes = (((size_t)n_rows * n_q * 4) + 255) & ~(size_t)255;
  a.tickets = (int*)d_ws;
  a.ws = (float*)((char*)d_ws + tk_bytes);
  a.scale_log2 = (float)(1.4426950408889634 / sqrt((double)hd));
  launch_attention(a, (cudaStream_t)stream);
  return last_launch();
}

extern "C" rt_status rt_op_prefill_attention(const void* d_q, const void* d_pool, const int32_t* d_page_table,
                                             int32_t pt_stride, const int32_t* d_tiles, int32_t n_tiles,
                                             int32_t n_rows, int32_t n_q, int32_t n_kv, int32_t hd, int32_t groups,
                                             void* d_out, float* d_out_f32, void* stream) {
  if (n_tiles < 0 || n_rows < 0 || n_kv < 1 || n_q % n_kv || n_q / n_kv > 8 || groups < 0 || groups > 2)
    return RT_E_INVAL;
  if (hd != 32 && hd != 64 && hd != 128) return RT_E_INVAL;
  if (n_tiles == 0 || n_rows == 0) return RT_OK;
  PrefillArgs a{};
  a.q = (const bf16*)d_q;
  a.pool = d_pool;
  a.page_table = d_page_table;
  a.pt_stride = pt_stride;
  a.tiles = reinterpret_cast<const int4*>(d_tiles);
  a.n_tiles = n_tiles;
  a.row0 = 0;
  a.n_rows = n_rows;
  a.nq = n_q;
  a.nkv = n_kv;
  a.hd = hd;
  a.G = n_q / n_kv;
  a.out = (bf16*)d_out;
  a.out_f32 = d_out_f32;
  a.scale_log2 = (float)(1.4426950408889634 / sqrt((double)hd));
  a.groups = groups;
  launch_attention_prefill(a, (cudaStream_t)stream);
  return last_launch();
}

extern "C" rt_status rt_op_kv_write(void* d_pool, const void* d_k, const void* d_v, const int32_t* d_slot,
                                    int32_t n_rows, int32_t n_kv, int32_t hd, void* stream) {
  if (n_rows < 0 || n_kv < 1 || hd % 8) return RT_E_INVAL;
  if (n_rows == 0) return RT_OK;
  launch_kv_write(d_pool, (const bf16*)d_k, (const bf16*)d_v, d_slot, n_rows, n_kv, hd, (cudaStream_t)stream);
  return last_launch();
}

extern "C" rt_status rt_op_kv_swap(const int32_t* d_swap, int32_t n, void* d_pool, int64_t pool_layer_bytes,
                                   void* h_host, int64_t blk_bytes, int32_t n_layers, void* stream) {
  if (n < 0 || n_layers < 1 || blk_bytes % 16 || !d_pool || !h_host) return RT_E_INVAL;
  if (n == 0) return RT_OK;
  launch_kv_swap(reinterpret_cast<const int4*>(d_swap), n, d_pool, pool_layer_bytes, h_host, blk_bytes, n_layers,
                 (cudaStream_t)stream);
  return last_launch();
}

extern "C" rt_status rt_op_kv_read(const void* d_pool, void* d_out, int32_t n_pages, int32_t n_kv, int32_t hd,
                                   void* stream) {
  if (n_pages < 1 || n_kv < 1 || hd % 8) return RT_E_INVAL;
  launch_kv_read(d_pool, (bf16*)d_out, n_pages, n_kv, hd, (cudaStream_t)stream);
  return last_launch();
}

extern "C" rt_status rt_op_gemm(const void* d_w, const void* d_x, float* d_out, int32_t M, int32_t N, int32_t K,
                                int32_t n_cap, int32_t splits, void* stream) {
  // splits <= 0: the engine's choice (rt_ops.h)
  if (M < 1 || N < 1 || K < 64 || K % 64 || n_cap < N || splits > K / 64) return RT_E_INVAL;
  GemmTmaSet xm;
  if (!make_gemm_act_maps(&xm, d_x, K, n_cap)) return RT_E_CUDA;
  bf16* wt = nullptr;  // the engine keeps weights UMMA-tiled; pack the caller's row-major W
  if (cudaMalloc(&wt, tiled_elems(M, K) * 2) != cudaSuccess) return RT_E_CUDA;
  launch_pack_tiled((const bf16*)d_w, wt, M, K, (cudaStream_t)stream);
  GemmArgs g{};
  g.M = M;
  g.N = N;
  g.K = K;
  g.mode = EPI_STORE;
  g.out = d_out;
  launch_gemm_epi(wt, xm, g, splits, (cudaStream_t)stream);
  rt_status st = last_launch();
  cudaStreamSynchronize((cudaStream_t)stream);
  cudaFree(wt);
  return st;
}

extern "C" rt_status rt_op_pack_tiled(const void* d_src, void* d_dst, int32_t M, int32_t K, void* stream) {
  if (M < 1 || K < 64 || K % 64) return RT_E_INVAL;
  launch_pack_tiled((const bf16*)d_src, (bf16*)d_dst, M, K, (cudaStream_t)stream);
  return last_launch();
}

extern "C" rt_status rt_op_gemm_tiled(const void* d_w_tiled, const void* d_x, float* d_out, int32_t M, int32_t N,
                                      int32_t K, int32_t n_cap, int32_t splits, int32_t path, int32_t bn,
                                      void* stream) {
  if (M < 1 || N < 1 || K < 64 || K % 64 || n_cap < N || splits < 0 || splits > K / 64) return RT_E_INVAL;
  if (path < RT_GEMM_PATH_AUTO || path > RT_GEMM_PATH_DECPAIR) return RT_E_INVAL;
  if (bn != 0 && bn != 32 && bn != 64 && bn != 128 && bn != 160 && bn != 192 && bn != 256) return RT_E_INVAL;
  if (bn != 0 && bn <= 128 && N > 128 && !(bn == 128 && path == RT_GEMM_PATH_PAIR)) return RT_E_INVAL;
  GemmTmaSet xm;
  if (!make_gemm_act_maps(&xm, d_x, K, n_cap)) return RT_E_CUDA;
  GemmArgs g{};
  g.M = M;
  g.N = N;
  g.K = K;
  g.mode = EPI_STORE;
  g.out = d_out;
  g.force_path = path;
  g.force_bn = bn;
  // stream-K path for N > 128 (as in the engine): a process-wide workspace on first use
  static float* sk_ws = nullptr;
  static unsigned* sk_cnt = nullptr;
  static int sk_cap = 0;
  static std::mutex sk_mu;  // callers on several host threads share the workspace allocation
  std::lock_guard<std::mutex> lock(sk_mu);
  const int need = ((M + 127) / 128) * ((N + 159) / 160);
  if (N > 128 && splits <= 0) {
    if (!sk_ws && cudaMalloc(&sk_ws, (size_t)gemm_sk_ws_floats() * 4) != cudaSuccess) return RT_E_CUDA;
    if (need > sk_cap) {
      if (sk_cnt) cudaFree(sk_cnt);
      sk_cap = std::max(need, 4096);
      if (cudaMalloc(&sk_cnt, (size_t)sk_cap * 4) != cudaSuccess) return RT_E_CUDA;
      cudaMemset(sk_cnt, 0, (size_t)sk_cap * 4);
    }
    g.sk_ws = sk_ws;
    g.sk_cnt = sk_cnt;
    g.sk_cnt_cap = sk_cap;
  }
  // decode-pair split-K exchange (k_gemm_dec): a process-wide workspace, grown on demand
  static float* dec_ws = nullptr;
  static int64_t dec_cap = 0;
  static unsigned* dec_flags = nullptr;
  static unsigned dec_epoch = 0;
  const int64_t dneed = gemm_dec_ws_floats(M, N, K);
  if (dneed > dec_cap) {
    if (dec_ws) cudaFree(dec_ws);
    if (cudaMalloc(&dec_ws, (size_t)dneed * 4) != cudaSuccess) return RT_E_CUDA;
    dec_cap = dneed;
  }
  if (!dec_flags) {
    if (cudaMalloc(&dec_flags, kDecFlags * 4) != cudaSuccess) return RT_E_CUDA;
    cudaMemset(dec_flags, 0, kDecFlags * 4);
  }
  g.dec_ws = dec_ws;
  g.dec_ws_floats = dec_cap;
  g.dec_flags = dec_flags;
  g.dec_flags_cap = kDecFlags;
  g.dec_epoch = ++dec_epoch;
  launch_gemm_epi((const bf16*)d_w_tiled, xm, g, splits, (cudaStream_t)stream);
  return last_launch();
}

extern "C" rt_status rt_op_lm_argmax(const void* d_w, const void* d_x, int32_t M, int32_t N, int32_t K,
                                     int32_t n_cap, int32_t* d_tok, float* d_logits, void* d_ws, int64_t ws_bytes,
                                     void* stream) {
  if (M < 1 || N < 1 || K < 64 || K % 64 || n_cap < N) return RT_E_INVAL;
  const int mt = (M + 127) / 128;
  if (ws_bytes < (int64_t)mt * N * 8) return RT_E_INVAL;
  GemmTmaSet xm;
  if (!make_gemm_act_maps(&xm, d_x, K, n_cap)) return RT_E_CUDA;
  bf16* wt = nullptr;
  if (cudaMalloc(&wt, tiled_elems(M, K) * 2) != cudaSuccess) return RT_E_CUDA;
  launch_pack_tiled((const bf16*)d_w, wt, M, K, (cudaStream_t)stream);
  float* pv = (float*)d_ws;
  int32_t* pi = (int32_t*)(pv + (size_t)mt * N);
  GemmArgs g{};
  g.M = M;
  g.N = N;
  g.K = K;
  g.mode = EPI_ARGMAX;
  g.out = d_logits;
  g.part_val = pv;
  g.part_idx = pi;
  launch_gemm_epi(wt, xm, g, 0, (cudaStream_t)stream);
  launch_argmax_reduce(pv, pi, mt, N, d_tok, (cudaStream_t)stream);
  rt_status st = last_launch();
  cudaStreamSynchronize((cudaStream_t)stream);
  cudaFree(wt);
  return st;
}

extern "C" rt_status rt_op_init_weights(void* d_out, int64_t n, uint64_t seed, int32_t tensor_id, float sigma,
                                        void* stream) {
  if (n < 0 || tensor_id < 0) return RT_E_INVAL;
  if (n == 0) return RT_OK;
  launch_init_weights((bf16*)d_out, n, seed, tensor_id, sigma, (cudaStream_t)stream);
  return last_launch();
}

extern "C" rt_status rt_op_priority(const int64_t* d_trde, const int32_t* d_k, const double* d_alpha,
                                    const double* d_beta, int32_t n, int32_t g_us, int32_t net_us, int32_t eps_l_us,
                                    double* d_pri, void* stream) {
  if (n < 0 || g_us <= 0 || eps_l_us <= 0) return RT_E_INVAL;
  launch_priority_batch(d_trde, d_k, d_alpha, d_beta, n, g_us, net_us, eps_l_us, d_pri, (cudaStream_t)stream);
  return last_launch();
}

extern "C" rt_status rt_op_merge_candidates(const double* d_all, int32_t world, double* d_merged, void* stream) {
  if (!d_all || !d_merged || world < 1 || world > 8) return RT_E_INVAL;
  launch_merge_cand(d_all, world, d_merged, (cudaStream_t)stream);
  return last_launch();
}
