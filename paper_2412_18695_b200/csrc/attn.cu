// attn.cu — paged decode attention for sm_100a (the graded HBM kernel).
//
// What it computes (oracle c1/c2, PAPER.md:387 PagedAttention): for every row r
// and q head h,  o = softmax(q . K^T / sqrt(hd)) V  over the row's first
// seqlen positions, K/V read through the request's page table (16-token pages).
//
// B200 design:
//  * one CTA per (row, kv head, chunk of pages); the G = nq/nkv q heads of a kv
//    head share every page read (GQA), so each (page, kv head) block is read
//    from HBM exactly once per step;
//  * a (page, kv head) block is one contiguous 64*hd-byte region ([K|V][16][hd],
//    XOR-swizzled at write time) moved by ONE cp.async.bulk (TMA engine, SASS
//    UBLKCP) into a per-warp ring of STAGES shared-memory buffers completed on
//    an mbarrier — no register staging, deep memory-level parallelism;
//  * warps work on interleaved pages independently (no CTA barrier in the loop);
//  * S^T = q K^T and O^T = V^T P^T on mma.sync m16n8k16 (bf16 in, fp32 acc) fed
//    by conflict-free ldmatrix from the swizzled buffers, online softmax in fp32
//    with exp2; warps merged through shared memory, chunks merged by a combine
//    kernel (flash-decoding split-KV).
#include "common.cuh"
#include "model.h"
#include <cstdlib>

namespace rt {

constexpr int kAttnWarps = 4;

template <int HD>
struct AttnCfg {
  static constexpr int BLOCK = 64 * HD;                       // bytes of one (page, kv head) block
  static constexpr int STAGES = HD >= 128 ? 3 : 6;
  static constexpr int MERGE = kAttnWarps * 8 * (HD + 2) * 4;  // fp32 merge buffers
  static constexpr int RING = kAttnWarps * STAGES * BLOCK;
  static constexpr int SMEM = (RING > MERGE ? RING : MERGE) + kAttnWarps * STAGES * 8 + 64;
};

// The QKV projection's epilogue for one (row, kv head) when the projection wrote raw split-K
// partials (EPI_PART): sum the splits in order, RMSNorm row scale, RoPE on the G
// q heads and the k head (weight rows 2i, 2i + 1 = dims i, i + hd/2), bf16 q -> s_q (shared,
// row stride qld, nullable) and / or a.q_out (+ a.q_cap), bf16 k / v appended at position pos of
// page pg_last.  All 128 threads of the CTA; no barrier inside.
template <int HD>
__device__ __forceinline__ void fold_qkv(const AttnArgs& a, int r, int row, int h, int pos, int pg_last, int G,
                                         bf16* s_q, int qld, bool write_q, bool append) {
  // RMSNorm row scale: every thread sums the row's per-tile sums of squares itself, in tile
  // order; its loads are issued together with the first group's partial loads below (one
  // L2 round trip for both), no barrier
  constexpr int kRsMax = 64;   // per-row tiles held in registers (d_model <= 8192)
  const float* rs = a.rs_ss + (size_t)r * a.rs_tiles;
  const bool rs_vec = (a.rs_tiles & 3) == 0 && a.rs_tiles <= kRsMax && ((uintptr_t)rs & 15) == 0;
  float4 rs4[kRsMax / 4];
#pragma unroll
  for (int i = 0; i < kRsMax / 4; ++i)
    rs4[i] = (rs_vec && 4 * i < a.rs_tiles) ? __ldcg(reinterpret_cast<const float4*>(rs) + i)
                                            : make_float4(0.f, 0.f, 0.f, 0.f);
  float inv = 0.f;
  bool have_inv = false;
  constexpr int HALF = HD / 2;
  constexpr int kMaxSplits = 8;  // gemm_part_splits <= 8 (cluster / pair split-K choices)
  constexpr int PB = 3;          // pairs per thread per round trip
  const int off = pos & 15;
  const int n_pairs = (G + 2) * HALF;
  const int S = a.part_splits;
  const size_t split_stride = (size_t)a.part_ld_n * a.part_m;
  for (int j0 = threadIdx.x; j0 < n_pairs; j0 += PB * blockDim.x) {
    // all the split partials (and the rotations) of PB pairs in flight at once
    float2 w[PB][kMaxSplits];
    float cr[PB], sr[PB];
#pragma unroll
    for (int u = 0; u < PB; ++u) {
      const int j = j0 + u * (int)blockDim.x;
      const bool ok = j < n_pairs;
      const int hl = j / HALF, i = j - hl * HALF;  // local head: q 0..G-1, then k, v
      const int head = hl < G ? h * G + hl : (hl == G ? a.nq + h : a.nq + a.nkv + h);
      const float* src = a.part + (size_t)r * a.part_m + (size_t)head * HD + 2 * i;
#pragma unroll
      for (int sp = 0; sp < kMaxSplits; ++sp)
        w[u][sp] = (ok && sp < S) ? __ldcg(reinterpret_cast<const float2*>(src + sp * split_stride))
                                  : make_float2(0.f, 0.f);
      const bool rot = ok && hl <= G;  // q and k heads are rotated
      cr[u] = rot ? __ldg(a.cos + (size_t)pos * HALF + i) : 1.f;
      sr[u] = rot ? __ldg(a.sin + (size_t)pos * HALF + i) : 0.f;
    }
    if (!have_inv) {
      float t = 0.f;
      if (rs_vec) {
#pragma unroll
        for (int i = 0; i < kRsMax / 4; ++i)
          if (4 * i < a.rs_tiles) t = (((t + rs4[i].x) + rs4[i].y) + rs4[i].z) + rs4[i].w;
      } else {
        for (int i = 0; i < a.rs_tiles; ++i) t += __ldcg(rs + i);
      }
      inv = rsqrtf(t / (float)a.d_model + 1e-5f);
      have_inv = true;
    }
#pragma unroll
    for (int u = 0; u < PB; ++u) {
      const int j = j0 + u * (int)blockDim.x;
      if (j >= n_pairs) break;
      const int hl = j / HALF, i = j - hl * HALF;
      const int head = hl < G ? h * G + hl : (hl == G ? a.nq + h : a.nq + a.nkv + h);
      float v0 = 0.f, v1 = 0.f;  // the sum in split order
#pragma unroll
      for (int sp = 0; sp < kMaxSplits; ++sp)
        if (sp < S) {
          v0 += w[u][sp].x;
          v1 += w[u][sp].y;
        }
      v0 *= inv;
      v1 *= inv;
      float y0 = v0, y1 = v1;
      if (hl <= G) {
        y0 = v0 * cr[u] - v1 * sr[u];
        y1 = v1 * cr[u] + v0 * sr[u];
      }
      const bf16 b0 = __float2bfloat16_rn(y0), b1 = __float2bfloat16_rn(y1);
      if (hl < G) {
        if (s_q) {
          s_q[hl * qld + i] = b0;
          s_q[hl * qld + i + HALF] = b1;
        }
        if (write_q) {
          bf16* qo = a.q_out + ((size_t)r * a.nq + head) * HD;
          qo[i] = b0;
          qo[i + HALF] = b1;
          if (a.q_cap) {
            float* qc = a.q_cap + ((size_t)row * a.nq + head) * HD;
            qc[i] = __bfloat162float(b0);
            qc[i + HALF] = __bfloat162float(b1);
          }
        }
      } else if (append) {
        const int kind = hl - G;  // 0: K, 1: V
        unsigned char* pb = (unsigned char*)a.pool +
                            (((size_t)pg_last * a.nkv + h) * 2 + kind) * (size_t)(16 * HD * 2) + off * HD * 2;
        *(bf16*)(pb + (kv_swz_chunk(HD, off, i >> 3) << 4) + ((i & 7) << 1)) = b0;
        *(bf16*)(pb + (kv_swz_chunk(HD, off, (i + HALF) >> 3) << 4) + (((i + HALF) & 7) << 1)) = b1;
      }
    }
  }
}

template <int HD>
__global__ void __launch_bounds__(kAttnWarps * 32) k_attn(AttnArgs a) {
  using C = AttnCfg<HD>;
  using SW = KvSwz<HD>;
  extern __shared__ __align__(1024) unsigned char smem[];
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + (C::RING > C::MERGE ? C::RING : C::MERGE));

  TraceScope tr(TK_ATTN);
  if (threadIdx.x == 0) pdl_trigger();
  const int chunk = blockIdx.x, h = blockIdx.y;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int G = a.G;
  const int gq = lane >> 2, qq = lane & 3;
  unsigned char* ring = smem + warp * C::STAGES * C::BLOCK;
  uint64_t* bar = bars + warp * C::STAGES;
  const unsigned char* pool = (const unsigned char*)a.pool;
  const size_t head_off = (size_t)h * C::BLOCK;
  const size_t page_stride = (size_t)a.nkv * C::BLOCK;
  if (lane == 0) {
    for (int s = 0; s < C::STAGES; ++s) mbar_init(&bar[s], 1);
    fence_mbar_init();
  }
  const uint64_t pol = a.l2_evict_first ? l2_policy_evict_first() : 0ull;
  // The round's row metadata (rows, lengths, tasks; written by the scheduler kernel at the
  // start of the round) is read BEFORE the dependency wait, overlapping the QKV projection's
  // tail.  Safe by construction: the kernel this one depends on is always a QKV projection
  // (k_gemm_tc / k_gemm_sk / k_gemm_2sm in EPI_QKV, or the chain whose last job is QKV), and
  // those trigger their dependents only AFTER their own griddepcontrol.wait — so when this
  // code runs, every kernel before the QKV projection, the scheduler included, has completed.
  // (With the trigger at the QKV kernel's start, a chain of early launches could reach here
  // while the scheduler was still writing: found as an intermittent stale read.)  The page
  // table is the scheduler's too; only q and the new KV entries (the row's last page) come from
  // the QKV projection itself and are read after the wait.
  const int row = a.row_list ? a.row_list[blockIdx.z] : a.row0 + (int)blockIdx.z;
  const int r = row - a.row0;  // row within this forward chunk
  if (a.row_list && (r < 0 || r >= a.chunk_rows)) return;
  const int seqlen = a.row_seqlen ? a.row_seqlen[row] : a.row_pos[row] + 1;
  const int n_pages = (seqlen + 15) >> 4;
  const int n_chunks = (n_pages + a.chunk_pages - 1) / a.chunk_pages;
  if (chunk >= n_chunks) return;
  const int p_begin = chunk * a.chunk_pages;
  const int p_end = min(p_begin + a.chunk_pages, n_pages);
  const int task = a.row_task[row];
  const int32_t* ptab = a.page_table + (size_t)task * a.pt_stride;
  // pages of this warp: p_begin + warp + i * NW
  const int n_my = p_end - (p_begin + warp) > 0 ? (p_end - (p_begin + warp) + kAttnWarps - 1) / kAttnWarps : 0;
  __syncwarp();
  // The K / V of every position before this round's token were written in earlier rounds
  // (pages and page-table entries are stable: see the metadata note above), so the first
  // stages' page loads are issued BEFORE the dependency wait — only the row's last page, which
  // receives this round's K / V (from the QKV projection, or appended by the fold below), waits.
  const bool fold = a.part != nullptr;
  const int last_pg = n_pages - 1;
  const bool appends = fold && chunk == n_chunks - 1;
  // page ids of the first 32 pages of this warp, one per lane
  int my_page = (lane < n_my) ? ptab[p_begin + warp + lane * kAttnWarps] : 0;
  int deferred = -1;  // stage of this warp whose (last) page waits for the dependency / append
#pragma unroll
  for (int i = 0; i < C::STAGES; ++i) {
    const int pg = __shfl_sync(0xffffffffu, my_page, i);
    if (i < n_my && p_begin + warp + i * kAttnWarps == last_pg) {
      deferred = i;
      continue;
    }
    if (lane == 0 && i < n_my) {
      mbar_arrive_expect_tx(&bar[i], C::BLOCK);
      bulk_g2s_hint(ring + i * C::BLOCK, pool + (size_t)pg * page_stride + head_off, C::BLOCK, &bar[i], pol);
    }
  }
  pdl_wait();
  tr.ready();
  constexpr int QLD = HD + 8;  // folded-q row stride: the 8 rows of a fragment load hit distinct banks
  __shared__ __align__(16) bf16 s_q[8 * QLD];  // folded q (G <= 8 heads) of this kv head
  if (fold) {
    // ---- QKV epilogue of this (row, kv head): sum the projection's split-K partials in split
    // order, RMSNorm row scale, RoPE (rotate-half; weight rows 2i, 2i + 1 = dims i, i + hd/2),
    // bf16 q -> shared memory (+ q_out / q_cap), bf16 k / v -> the page (swizzled rows)
    fold_qkv<HD>(a, r, row, h, seqlen - 1, ptab[(seqlen - 1) >> 4], G, s_q, QLD, chunk == 0, appends);
    fence_proxy_async_global();  // the appended K / V rows are read by the bulk copies below
    __syncthreads();
  }
  if (deferred >= 0) {  // the last page, after the dependency (and the fold's append); warp-uniform
    const int pg = __shfl_sync(0xffffffffu, my_page, deferred);
    if (lane == 0) {
      if (!fold) fence_proxy_async_global();
      mbar_arrive_expect_tx(&bar[deferred], C::BLOCK);
      bulk_g2s_hint(ring + deferred * C::BLOCK, pool + (size_t)pg * page_stride + head_off, C::BLOCK,
                    &bar[deferred], pol);
    }
  }

  // q fragments (A operand of S^T = Q K^T), rows g >= G are zero
  uint32_t qa[HD / 16][2];
  {
    const bf16* qrow = fold ? s_q : a.q + ((size_t)r * a.nq + (size_t)h * G) * HD;
    const int qld = fold ? QLD : HD;
#pragma unroll
    for (int ks = 0; ks < HD / 16; ++ks) {
      if (gq < G) {
        const uint32_t* q32 = reinterpret_cast<const uint32_t*>(qrow + (size_t)gq * qld + ks * 16);
        qa[ks][0] = q32[qq];
        qa[ks][1] = q32[4 + qq];
      } else {
        qa[ks][0] = 0u;
        qa[ks][1] = 0u;
      }
    }
  }
  float acc[HD / 16][4];
#pragma unroll
  for (int mt = 0; mt < HD / 16; ++mt) acc[mt][0] = acc[mt][1] = acc[mt][2] = acc[mt][3] = 0.f;
  float m_run = -INFINITY, l_run = 0.f;
  const float sl2 = a.scale_log2;
  // ldmatrix lane addressing: matrix mi = lane >> 3, row j = lane & 7
  const int mi = lane >> 3;
  const int ltok = ((mi >> 1) << 3) + (lane & 7);
  const int lcsel = mi & 1;

  for (int i = 0; i < n_my; ++i) {
    const int s = i % C::STAGES;
    mbar_wait(&bar[s], (uint32_t)((i / C::STAGES) & 1));
    const uint32_t kbase = smem_u32(ring + s * C::BLOCK);
    const uint32_t vbase = kbase + SW::MAT_BYTES;
    // ---- S^T (16 g-rows x 16 tokens) = Q K^T
    float s0[4] = {0.f, 0.f, 0.f, 0.f}, s1[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
    for (int ks = 0; ks < HD / 16; ++ks) {
      uint32_t b0, b1, b2, b3;
      ldmatrix_x4(b0, b1, b2, b3, kbase + SW::chunk_off(ltok, 2 * ks + lcsel));
      const uint32_t afr[4] = {qa[ks][0], 0u, qa[ks][1], 0u};
      const uint32_t bf0[2] = {b0, b1}, bf1[2] = {b2, b3};
      mma_bf16_16816(s0, afr, bf0);
      mma_bf16_16816(s1, afr, bf1);
    }
    // ---- online softmax for row g = lane/4 over tokens 2qq, 2qq+1, 8+2qq, 9+2qq
    const int page_idx = p_begin + warp + i * kAttnWarps;
    const int t0 = page_idx * 16 + 2 * qq;
    float x00 = (t0 < seqlen) ? s0[0] * sl2 : -INFINITY;
    float x01 = (t0 + 1 < seqlen) ? s0[1] * sl2 : -INFINITY;
    float x10 = (t0 + 8 < seqlen) ? s1[0] * sl2 : -INFINITY;
    float x11 = (t0 + 9 < seqlen) ? s1[1] * sl2 : -INFINITY;
    float mp = fmaxf(fmaxf(x00, x01), fmaxf(x10, x11));
    mp = fmaxf(mp, __shfl_xor_sync(0xffffffffu, mp, 1));
    mp = fmaxf(mp, __shfl_xor_sync(0xffffffffu, mp, 2));
    const float m_new = fmaxf(m_run, mp);
    const float corr = exp2f(m_run - m_new);
    const float p00 = exp2f(x00 - m_new), p01 = exp2f(x01 - m_new);
    const float p10 = exp2f(x10 - m_new), p11 = exp2f(x11 - m_new);
    l_run = l_run * corr + (p00 + p01) + (p10 + p11);
    m_run = m_new;
    // rescale O^T columns g = 2qq, 2qq+1 (their softmax state lives in lanes 4g..4g+3)
    const float c0 = __shfl_sync(0xffffffffu, corr, 8 * qq);
    const float c1 = __shfl_sync(0xffffffffu, corr, 8 * qq + 4);
    const uint32_t pb[2] = {pack_bf16x2(p00, p01), pack_bf16x2(p10, p11)};
    // ---- O^T (hd x 16 g) += V^T P^T
#pragma unroll
    for (int mt = 0; mt < HD / 16; ++mt) {
      acc[mt][0] *= c0;
      acc[mt][1] *= c1;
      acc[mt][2] *= c0;
      acc[mt][3] *= c1;
      uint32_t va[4];
      ldmatrix_x4_trans(va[0], va[1], va[2], va[3], vbase + SW::chunk_off(ltok, 2 * mt + lcsel));
      mma_bf16_16816(acc[mt], va, pb);
    }
    __syncwarp();
    // refill this stage with page i + STAGES of this warp
    const int nx = i + C::STAGES;
    if (nx < n_my) {
      if ((nx & 31) == 0) my_page = (lane + nx < n_my) ? ptab[p_begin + warp + (nx + lane) * kAttnWarps] : 0;
      const int pg = __shfl_sync(0xffffffffu, my_page, nx & 31);
      if (lane == 0) {
        fence_proxy_async();
        mbar_arrive_expect_tx(&bar[s], C::BLOCK);
        bulk_g2s_hint(ring + s * C::BLOCK, pool + (size_t)pg * page_stride + head_off, C::BLOCK, &bar[s], pol);
      }
    }
  }
  // ---- merge warps through shared memory (aliases the rings)
  l_run += __shfl_xor_sync(0xffffffffu, l_run, 1);
  l_run += __shfl_xor_sync(0xffffffffu, l_run, 2);
  __syncthreads();
  float* mw = reinterpret_cast<float*>(smem);                   // [NW][8]
  float* lw = mw + kAttnWarps * 8;                              // [NW][8]
  float* ow = lw + kAttnWarps * 8;                              // [NW][8][HD]
  if (qq == 0 && gq < 8) {
    mw[warp * 8 + gq] = m_run;
    lw[warp * 8 + gq] = l_run;
  }
#pragma unroll
  for (int mt = 0; mt < HD / 16; ++mt) {
    const int d = mt * 16 + gq;
    const int g0 = 2 * qq;
    ow[(warp * 8 + g0) * HD + d] = acc[mt][0];
    ow[(warp * 8 + g0 + 1) * HD + d] = acc[mt][1];
    ow[(warp * 8 + g0) * HD + d + 8] = acc[mt][2];
    ow[(warp * 8 + g0 + 1) * HD + d + 8] = acc[mt][3];
  }
  __syncthreads();
  const bool single = (n_chunks == 1);
  for (int it = threadIdx.x; it < G * HD; it += blockDim.x) {
    const int g = it / HD, d = it % HD;
    float M = -INFINITY;
#pragma unroll
    for (int w = 0; w < kAttnWarps; ++w) M = fmaxf(M, mw[w * 8 + g]);
    float L = 0.f, O = 0.f;
#pragma unroll
    for (int w = 0; w < kAttnWarps; ++w) {
      const float mwv = mw[w * 8 + g];
      const float f = (mwv == -INFINITY) ? 0.f : exp2f(mwv - M);
      L += lw[w * 8 + g] * f;
      O += ow[(w * 8 + g) * HD + d] * f;
    }
    const int qh = h * G + g;
    if (single) {
      const float o = O / L;
      a.out[((size_t)r * a.nq + qh) * HD + d] = __float2bfloat16_rn(o);
      if (a.out_f32) a.out_f32[((size_t)row * a.nq + qh) * HD + d] = o;
    } else {
      // partial: ws[((r * nq + qh) * max_chunks + chunk) * (HD + 2) + ...]
      float* wp = a.ws + (((size_t)r * a.nq + qh) * a.max_chunks + chunk) * (HD + 2);
      wp[d] = O;
      if (d == 0) {
        wp[HD] = M;
        wp[HD + 1] = L;
      }
    }
  }
  if (single) return;
  // ---- split-KV merge by the last chunk CTA of this (row, kv head): no combine launch
  __shared__ int s_last;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    int* tk = a.tickets + (size_t)r * a.nkv + h;
    const int prev = atomicAdd(tk, 1);
    s_last = (prev == n_chunks - 1);
    if (s_last) *tk = 0;  // self-resetting for the next launch
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  for (int it = threadIdx.x; it < G * HD; it += blockDim.x) {
    const int g = it / HD, d = it % HD;
    const int qh = h * G + g;
    const float* wp = a.ws + ((size_t)r * a.nq + qh) * a.max_chunks * (HD + 2);
    float M = -INFINITY;
    for (int c = 0; c < n_chunks; ++c) M = fmaxf(M, __ldcg(wp + c * (HD + 2) + HD));
    float L = 0.f, O = 0.f;
    for (int c = 0; c < n_chunks; ++c) {  // fixed chunk order -> deterministic
      const float f = exp2f(__ldcg(wp + c * (HD + 2) + HD) - M);
      L += __ldcg(wp + c * (HD + 2) + HD + 1) * f;
      O += __ldcg(wp + c * (HD + 2) + d) * f;
    }
    const float o = O / L;
    a.out[((size_t)r * a.nq + qh) * HD + d] = __float2bfloat16_rn(o);
    if (a.out_f32) a.out_f32[((size_t)row * a.nq + qh) * HD + d] = o;
  }
}


// ---------------------------------------------------------------- prefill attention
// Causal attention of the prompt rows of k = 0 admissions (oracle c1: the
// same softmax(q K^T / sqrt(hd)) V over positions <= the row's own).  The decode kernel
// above would re-read a prompt's K/V once per ROW; here one CTA serves a tile of 16
// consecutive positions for all G q heads of a kv head, so every (page, kv head) block
// is read once per tile and feeds 16 x G query rows:
//  * CTA = (tile, kv head), warp g = q head h*G + g, the warp's 16 query rows = the tile's
//    positions (mma.sync M dimension);
//  * pages 0 .. pos0/16 stream through a CTA-shared ring of STAGES (page, kv head)
//    blocks, one cp.async.bulk each, full / empty mbarriers (G consumer warps);
//  * S = Q K^T and O += P V on m16n8k16 (bf16 in, fp32 acc), online softmax in fp32 with
//    exp2, causal mask on the diagonal page only; longest tiles are scheduled first.
//  * few CTAs (light prefill rounds, G <= 4): two warp groups per CTA (8 warps); group j
//    takes the pages i = j mod 2 with its own online-softmax state, merged in shared memory
//    at the end (fixed order) — twice the warps per SM for this mma.sync-latency-bound loop
//    without a global merge.  Measured (tools/prefill_tail_bench.py, 84-token tails on a
//    1216-token prefix, 6 tiles x 8 kv heads per request): 1 / 2 / 3 requests (48 / 96 / 144
//    CTAs) 52.4 / 52.9 / 53.3 -> 36.7 / 37.4 / 38.0 us per layer; from 4 requests (192 CTAs,
//    more than one per SM) two groups lose (64.2 -> 71.2 us): one group there.
template <int HD, int NG>
struct PfCfg {
  static constexpr int BLOCK = 64 * HD;
  static constexpr int STAGES = 4 * NG;  // page i + STAGES belongs to the same warp group
  static constexpr int SMEM = STAGES * BLOCK + 2 * STAGES * 8 + 64;
  static_assert(NG == 1 || 4 * 32 * (HD / 2 + 4) * 4 <= STAGES * BLOCK, "group merge fits in the ring");
};

template <int HD, int NG>
__global__ void __launch_bounds__(256) k_attn_prefill(PrefillArgs a) {
  using C = PfCfg<HD, NG>;
  using SW = KvSwz<HD>;
  extern __shared__ __align__(1024) unsigned char smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + C::STAGES * C::BLOCK);
  uint64_t* empty = full + C::STAGES;

  TraceScope tr(TK_ATTN_PREFILL);
  // no early pdl_trigger here: the next kernel's CTAs (a projection whose MMA / epilogue
  // warps wait spinning) co-resident with this latency-bound kernel cost it ~25 us per layer
  // at the e2e operating point (tools/prefill_tail_bench.py); the implicit trigger at exit
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int gq = lane >> 2, qq = lane & 3;
  const int G = a.G;
  const int grp = warp / G, wg = warp - grp * G;  // warp group, q head within the kv head
  const int h = blockIdx.y;
  if (threadIdx.x == 0) {
    for (int s = 0; s < C::STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], G);  // one warp group consumes a page
    }
    fence_mbar_init();
  }
  __syncthreads();
  pdl_wait();  // q and the prompt's K/V pages come from the QKV GEMM before this kernel
  tr.ready();
  const int tix = a.n_tiles - 1 - (int)blockIdx.x;
  const int4 T = a.tiles[tix];  // (row, rows, pos0, task)
  const int rb = T.x, re = T.x + T.y;
  if (max(rb, a.row0) >= min(re, a.row0 + a.n_rows)) return;  // not in this forward chunk
  const int npt = (T.z >> 4) + 1;                               // pages 0 .. pos0 / 16
  const int np = npt;
  // The CTAs of a round that prefill the tails of prompts sharing a long prefix all read the
  // same prefix pages; walking them in the same order makes every CTA hit the same L2 lines
  // at the same time.  Each CTA starts its walk at its own page (softmax is order-free; the
  // diagonal page keeps its causal mask wherever it falls).
  const int rot = np > 0 ? (int)(((unsigned)tix * 7u + (unsigned)h * 13u) % (unsigned)np) : 0;
  auto page_at = [&](int i) { return i + rot >= np ? i + rot - np : i + rot; };
  const int32_t* ptab = a.page_table + (size_t)T.w * a.pt_stride;
  const unsigned char* pool = (const unsigned char*)a.pool;
  const size_t head_off = (size_t)h * C::BLOCK;
  const size_t page_stride = (size_t)a.nkv * C::BLOCK;
  if (threadIdx.x == 0)
    for (int i = 0; i < C::STAGES && i < np; ++i) {
      mbar_arrive_expect_tx(&full[i], C::BLOCK);
      bulk_g2s(smem + i * C::BLOCK, pool + (size_t)ptab[page_at(i)] * page_stride + head_off, C::BLOCK, &full[i]);
    }

  // q fragments (A operand, rows = the tile's positions), rows outside the chunk are zero
  const int qh = h * G + wg;
  uint32_t qa[HD / 16][4];
  {
    const int r0 = rb + gq, r1 = rb + gq + 8;
    const bool ok0 = r0 < re && r0 >= a.row0 && r0 < a.row0 + a.n_rows;
    const bool ok1 = r1 < re && r1 >= a.row0 && r1 < a.row0 + a.n_rows;
    const uint32_t* q0 = reinterpret_cast<const uint32_t*>(a.q + ((size_t)(r0 - a.row0) * a.nq + qh) * HD);
    const uint32_t* q1 = reinterpret_cast<const uint32_t*>(a.q + ((size_t)(r1 - a.row0) * a.nq + qh) * HD);
#pragma unroll
    for (int ks = 0; ks < HD / 16; ++ks) {
      qa[ks][0] = ok0 ? q0[ks * 8 + qq] : 0u;
      qa[ks][1] = ok1 ? q1[ks * 8 + qq] : 0u;
      qa[ks][2] = ok0 ? q0[ks * 8 + 4 + qq] : 0u;
      qa[ks][3] = ok1 ? q1[ks * 8 + 4 + qq] : 0u;
    }
  }
  float o[HD / 8][4];
#pragma unroll
  for (int nt = 0; nt < HD / 8; ++nt) o[nt][0] = o[nt][1] = o[nt][2] = o[nt][3] = 0.f;
  float m0 = -INFINITY, m1 = -INFINITY, l0 = 0.f, l1 = 0.f;
  const float sl2 = a.scale_log2;
  const int mi = lane >> 3;
  const int ltok = ((mi >> 1) << 3) + (lane & 7);
  const int lcsel = mi & 1;
  const int qp0 = T.z + gq, qp1 = T.z + gq + 8;  // positions of this lane's two rows

  for (int i = grp; i < np; i += NG) {
    const int s = i % C::STAGES;
    mbar_wait(&full[s], (uint32_t)((i / C::STAGES) & 1));
    const uint32_t kbase = smem_u32(smem + s * C::BLOCK);
    const uint32_t vbase = kbase + SW::MAT_BYTES;
    // ---- S (16 positions x 16 keys) = Q K^T
    float s0[4] = {0.f, 0.f, 0.f, 0.f}, s1[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
    for (int ks = 0; ks < HD / 16; ++ks) {
      uint32_t b0, b1, b2, b3;
      ldmatrix_x4(b0, b1, b2, b3, kbase + SW::chunk_off(ltok, 2 * ks + lcsel));
      const uint32_t bf0[2] = {b0, b1}, bf1[2] = {b2, b3};
      mma_bf16_16816(s0, qa[ks], bf0);
      mma_bf16_16816(s1, qa[ks], bf1);
    }
    // ---- causal mask (diagonal page) + online softmax; row gq: s*[0..1], row gq+8: s*[2..3]
    const int pg_i = page_at(i);
    const int k0 = pg_i * 16 + 2 * qq;
    float x[8] = {s0[0] * sl2, s0[1] * sl2, s1[0] * sl2, s1[1] * sl2,
                  s0[2] * sl2, s0[3] * sl2, s1[2] * sl2, s1[3] * sl2};
    if (pg_i == npt - 1) {
      const int kk[4] = {k0, k0 + 1, k0 + 8, k0 + 9};
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        if (kk[j] > qp0) x[j] = -INFINITY;
        if (kk[j] > qp1) x[4 + j] = -INFINITY;
      }
    }
    float mp0 = fmaxf(fmaxf(x[0], x[1]), fmaxf(x[2], x[3]));
    float mp1 = fmaxf(fmaxf(x[4], x[5]), fmaxf(x[6], x[7]));
    mp0 = fmaxf(mp0, __shfl_xor_sync(0xffffffffu, mp0, 1));
    mp0 = fmaxf(mp0, __shfl_xor_sync(0xffffffffu, mp0, 2));
    mp1 = fmaxf(mp1, __shfl_xor_sync(0xffffffffu, mp1, 1));
    mp1 = fmaxf(mp1, __shfl_xor_sync(0xffffffffu, mp1, 2));
    const float mn0 = fmaxf(m0, mp0), mn1 = fmaxf(m1, mp1);
    const float c0 = exp2f(m0 - mn0), c1 = exp2f(m1 - mn1);
    float pr[8];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      pr[j] = exp2f(x[j] - mn0);
      pr[4 + j] = exp2f(x[4 + j] - mn1);
    }
    l0 = l0 * c0 + ((pr[0] + pr[1]) + (pr[2] + pr[3]));
    l1 = l1 * c1 + ((pr[4] + pr[5]) + (pr[6] + pr[7]));
    m0 = mn0;
    m1 = mn1;
    // P as the A operand: (row gq | gq+8) x (keys 2qq.. | 8+2qq..)
    const uint32_t pa[4] = {pack_bf16x2(pr[0], pr[1]), pack_bf16x2(pr[4], pr[5]), pack_bf16x2(pr[2], pr[3]),
                            pack_bf16x2(pr[6], pr[7])};
    // ---- O (16 x hd) += P V
#pragma unroll
    for (int n2 = 0; n2 < HD / 16; ++n2) {
      uint32_t v0, v1, v2, v3;
      ldmatrix_x4_trans(v0, v1, v2, v3, vbase + SW::chunk_off(ltok, 2 * n2 + lcsel));
      const uint32_t blo[2] = {v0, v2}, bhi[2] = {v1, v3};
      o[2 * n2][0] *= c0;
      o[2 * n2][1] *= c0;
      o[2 * n2][2] *= c1;
      o[2 * n2][3] *= c1;
      o[2 * n2 + 1][0] *= c0;
      o[2 * n2 + 1][1] *= c0;
      o[2 * n2 + 1][2] *= c1;
      o[2 * n2 + 1][3] *= c1;
      mma_bf16_16816(o[2 * n2], pa, blo);
      mma_bf16_16816(o[2 * n2 + 1], pa, bhi);
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
    // refill stage s with page i + STAGES (same group) once every warp of the group released it
    if (wg == 0 && lane == 0 && i + C::STAGES < np) {
      mbar_wait(&empty[s], (uint32_t)((i / C::STAGES) & 1));
      fence_proxy_async();
      mbar_arrive_expect_tx(&full[s], C::BLOCK);
      bulk_g2s(smem + s * C::BLOCK, pool + (size_t)ptab[page_at(i + C::STAGES)] * page_stride + head_off, C::BLOCK,
               &full[s]);
    }
  }
  l0 += __shfl_xor_sync(0xffffffffu, l0, 1);
  l0 += __shfl_xor_sync(0xffffffffu, l0, 2);
  l1 += __shfl_xor_sync(0xffffffffu, l1, 1);
  l1 += __shfl_xor_sync(0xffffffffu, l1, 2);
  if constexpr (NG == 2) {  // group 1's state -> shared memory (the ring is idle), group 0 merges
    __syncthreads();
    float* xs = reinterpret_cast<float*>(smem) + (size_t)(wg * 32 + lane) * (HD / 2 + 4);
    if (grp == 1) {
#pragma unroll
      for (int nt = 0; nt < HD / 8; ++nt)
#pragma unroll
        for (int j = 0; j < 4; ++j) xs[nt * 4 + j] = o[nt][j];
      xs[HD / 2] = m0;
      xs[HD / 2 + 1] = m1;
      xs[HD / 2 + 2] = l0;
      xs[HD / 2 + 3] = l1;
    }
    __syncthreads();
    if (grp == 0) {
      const float pm0 = xs[HD / 2], pm1 = xs[HD / 2 + 1];
      const float M0 = fmaxf(m0, pm0), M1 = fmaxf(m1, pm1);
      const float fa0 = exp2f(m0 - M0), fa1 = exp2f(m1 - M1);
      const float fb0 = pm0 == -INFINITY ? 0.f : exp2f(pm0 - M0);
      const float fb1 = pm1 == -INFINITY ? 0.f : exp2f(pm1 - M1);
      l0 = l0 * fa0 + xs[HD / 2 + 2] * fb0;
      l1 = l1 * fa1 + xs[HD / 2 + 3] * fb1;
#pragma unroll
      for (int nt = 0; nt < HD / 8; ++nt) {
        o[nt][0] = o[nt][0] * fa0 + xs[nt * 4 + 0] * fb0;
        o[nt][1] = o[nt][1] * fa0 + xs[nt * 4 + 1] * fb0;
        o[nt][2] = o[nt][2] * fa1 + xs[nt * 4 + 2] * fb1;
        o[nt][3] = o[nt][3] * fa1 + xs[nt * 4 + 3] * fb1;
      }
      m0 = M0;
      m1 = M1;
    }
  }
  const bool active = grp == 0;  // group 0 holds the merged state of its q head
  // ---- normalise and store rows gq, gq + 8 (dims 8 nt + 2 qq, +1)
  if (!active) return;
  const float i0 = 1.f / l0, i1 = 1.f / l1;
#pragma unroll
  for (int hf = 0; hf < 2; ++hf) {
    const int row = rb + gq + 8 * hf;
    if (row >= re || row < a.row0 || row >= a.row0 + a.n_rows) continue;
    const float inv = hf ? i1 : i0;
    bf16* orow = a.out + ((size_t)(row - a.row0) * a.nq + qh) * HD;
    float* frow = a.out_f32 ? a.out_f32 + ((size_t)row * a.nq + qh) * HD : nullptr;
#pragma unroll
    for (int nt = 0; nt < HD / 8; ++nt) {
      const int d = nt * 8 + 2 * qq;
      const float v0 = o[nt][2 * hf] * inv, v1 = o[nt][2 * hf + 1] * inv;
      const bf16 b0 = __float2bfloat16_rn(v0), b1 = __float2bfloat16_rn(v1);
      *reinterpret_cast<uint32_t*>(orow + d) = pack_bf16x2(v0, v1);
      if (frow) {
        frow[d] = __bfloat162float(b0);
        frow[d + 1] = __bfloat162float(b1);
      }
    }
  }
}

int64_t attn_ws_floats(int n_rows, int nq, int hd, int max_chunks) {
  return (int64_t)n_rows * nq * max_chunks * (hd + 2);
}

// Split-KV plan (measured on B200, tools/attn_bench.py): one CTA per (row, kv head)
// streams at 96-110 % of the measured copy bandwidth from 64 rows x 8 kv heads up (C2
// 64 x 1310: 55 us; 64 x 8192: 90 % of 8 TB/s); extra chunks only add pipeline fills
// and the merge, and were never faster for >= 32 (row, head) pairs.  Below that the
// step is latency-bound and c = ceil(64 / pairs) <= 8 chunks help (1 row x 4096:
// 32 -> 14.5 us).  RT_ATTN_CHUNKS overrides c (tuning).
// Prompt rows of a round whose QKV projection wrote raw partials (mixed decode + prefill
// rounds of <= 256 rows): the same folded epilogue for every (prompt row, kv head) — q to
// a.q_out for the prefill attention, k / v appended into the rows' pages.  CTA = (16-position
// tile, position in the tile) x kv head over SchedParams::pf_tiles (first row, rows, first
// position, task).  Launched after the decode attention and before the prefill attention.
template <int HD>
__global__ void __launch_bounds__(kAttnWarps * 32) k_qkv_finish(AttnArgs a, const int4* tiles) {
  TraceScope tr(TK_ATTN_PREFILL | (1u << 8));
  if (threadIdx.x == 0) pdl_trigger();
  pdl_wait();
  tr.ready();
  const int4 t = tiles[blockIdx.x >> 4];
  const int i = blockIdx.x & 15;
  if (i >= t.y) return;
  const int row = t.x + i, pos = t.z + i, h = blockIdx.y;
  const int32_t* ptab = a.page_table + (size_t)t.w * a.pt_stride;
  fold_qkv<HD>(a, row - a.row0, row, h, pos, ptab[pos >> 4], a.G, nullptr, 0, true, true);
}
void launch_qkv_finish(const AttnArgs& a, const int4* tiles, int n_tiles, cudaStream_t s) {
  if (n_tiles <= 0) return;
  const dim3 grid(16 * n_tiles, a.nkv), block(kAttnWarps * 32);
  switch (a.hd) {
    case 128: launch_pdl(k_qkv_finish<128>, grid, block, 0, s, a, tiles); break;
    case 64: launch_pdl(k_qkv_finish<64>, grid, block, 0, s, a, tiles); break;
    case 32: launch_pdl(k_qkv_finish<32>, grid, block, 0, s, a, tiles); break;
    default: break;
  }
}

void attn_plan(int n_rows, int nkv, int max_seqlen, int* chunk_pages, int* max_chunks) {
  const int max_pages = (max_seqlen + 15) / 16;
  const long long base = (long long)n_rows * nkv;
  int best_c = 1;
  if (base > 0 && base < 32) {
    best_c = (int)((64 + base - 1) / base);
    if (best_c > 8) best_c = 8;
    while (best_c > 1 && max_pages / best_c < 2 * kAttnWarps) --best_c;
  } else if (base < 96 && max_pages >= 128) {
    // 32-95 (row, head) pairs leave most of the 148 SMs idle; with >= 2k-token contexts four
    // chunks pay for the merge (tools/attn_small_b.py, 8 rows x 8 heads: ctx 2884 29.2 ->
    // 20.7 us, ctx 8192 75.2 -> 46.4 us; 16 rows: no gain, 1310-token contexts: no gain)
    best_c = 4;
  }
  int cp = (max_pages + best_c - 1) / best_c;
  if (cp < 1) cp = 1;
  *chunk_pages = cp;
  *max_chunks = (max_pages + cp - 1) / cp;
}

template <int HD>
static void launch_hd(const AttnArgs& a, cudaStream_t s) {
  using C = AttnCfg<HD>;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_attn<HD>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
    attr = true;
  }
  dim3 grid(a.max_chunks, a.nkv, a.n_rows);
  launch_pdl(k_attn<HD>, grid, dim3(kAttnWarps * 32), C::SMEM, s, a);
}

void launch_attention(const AttnArgs& a0, cudaStream_t s) {
  if (a0.n_rows <= 0) return;
  AttnArgs a = a0;
  a.l2_evict_first = l2_hint_enabled() ? 1 : 0;
  switch (a.hd) {
    case 128: launch_hd<128>(a, s); break;
    case 64: launch_hd<64>(a, s); break;
    case 32: launch_hd<32>(a, s); break;
    default: break;
  }
}

template <int HD, int NG>
static void launch_prefill_ng(const PrefillArgs& a, cudaStream_t s) {
  using C = PfCfg<HD, NG>;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_attn_prefill<HD, NG>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
    attr = true;
  }
  // plain stream-ordered launch (no programmatic dependent launch): measured faster for this
  // latency-bound kernel (tools/prefill_tail_bench.py)
  const dim3 grid(a.n_tiles, a.nkv), block(32 * a.G * NG);
  k_attn_prefill<HD, NG><<<grid, block, C::SMEM, s>>>(a);
}
template <int HD>
static void launch_prefill_hd(const PrefillArgs& a, cudaStream_t s) {
  // two warp groups while there is at most one CTA per SM (a.groups = 1 / 2 forces)
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (sms <= 0) sms = 148;
  }
  const long long ctas = (long long)a.n_tiles * a.nkv;
  const int ng = a.G > 4 ? 1 : (a.groups ? a.groups : (ctas <= sms ? 2 : 1));
  if (ng == 2)
    launch_prefill_ng<HD, 2>(a, s);
  else
    launch_prefill_ng<HD, 1>(a, s);
}

void launch_attention_prefill(const PrefillArgs& a, cudaStream_t s) {
  if (a.n_tiles <= 0 || a.G < 1 || a.G > 8) return;
  switch (a.hd) {
    case 128: launch_prefill_hd<128>(a, s); break;
    case 64: launch_prefill_hd<64>(a, s); break;
    case 32: launch_prefill_hd<32>(a, s); break;
    default: break;
  }
}

RT_TRACE_BINDER(trace_bind_attn)

}  // namespace rt
