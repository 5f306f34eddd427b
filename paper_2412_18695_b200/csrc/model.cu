// model.cu — elementwise / row kernels of the Llama decode step.
//
// The GEMMs (gemm_tc.cu) write fp32 split-K partials; the "epilogue" kernels
// here reduce the partials and apply the fused elementwise work the oracle's c1
// definition places between two GEMMs (RMSNorm, RoPE + KV append, SwiGLU,
// residual add), rounding to bf16 exactly at the materialisation points of
// DESIGN.md (GEMM inputs, q after RoPE, stored K/V).  The residual stream x is
// fp32.
#include "common.cuh"
#include "model.h"
#include <algorithm>

namespace rt {

// ------------------------------------------------------- counter-based init
// DESIGN.md AMB-15: u = splitmix64(seed ^ (tensor_id << 40) ^ idx);
// w = bf16_rne(fp32(((u >> 40) * 2^-24 - 0.5)) * c), c = fp32(2 sqrt(3) sigma)
__device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
  uint64_t z = x + 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

__global__ void k_init_weights(bf16* out, int64_t n, uint64_t seed, int32_t tensor_id, float c) {
  const uint64_t key = seed ^ ((uint64_t)tensor_id << 40);
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t u = splitmix64(key ^ (uint64_t)i);
    const float r = __fsub_rn(__fmul_rn((float)(uint32_t)(u >> 40), 5.9604644775390625e-08f), 0.5f);
    out[i] = __float2bfloat16_rn(__fmul_rn(r, c));
  }
}


// ------------------------------------------- UMMA-tiled weight layout
// A [M, K] weight is stored as contiguous 128 x 64 bf16 tiles (16 KiB), tile (mt, kb)
// at index mt * KB + kb, each tile in the SW128 K-major smem image: row r, 16-byte
// chunk c stored at chunk c ^ (r & 7).  One cp.async.bulk of 16 KiB per k-block
// lands a ready UMMA operand; a CTA streams one contiguous HBM range.
// Logical row of tiled row p, or -1 for a zero pad row.  The GEMM epilogues combine PAIRS
// of rows, which the layout puts in adjacent rows (adjacent TMEM lanes -> one warp
// shuffle, no shared-memory exchange):
//   gu_ff > 0   (W_gate_up, [2 ff, d]): tile t holds features [64 t, 64 t + 64), physical
//               row 2k = gate of feature 64 t + k, row 2k + 1 = its up row;
//   rope_hd > 0 (W_qkv): inside every head block of rope_hd rows, physical row 2k = dim k,
//               row 2k + 1 = dim k + rope_hd / 2 (the rotate-half partner).
__device__ __forceinline__ int64_t tiled_logical_row(int64_t p, int M, int gu_ff, int rope_hd) {
  if (gu_ff > 0) {
    const int64_t j = 64 * (p >> 7) + ((p & 127) >> 1);
    if (j >= gu_ff) return -1;
    return (p & 1) ? (int64_t)gu_ff + j : j;
  }
  if (p >= M) return -1;
  if (rope_hd > 0) {
    const int64_t h = p / rope_hd, r = p % rope_hd;
    return h * rope_hd + (r >> 1) + ((r & 1) ? rope_hd / 2 : 0);
  }
  return p;
}
// element i of the tiled buffer -> (physical row p, logical column col)
__device__ __forceinline__ void tiled_coords(int64_t i, int KB, int64_t* p, int* col) {
  const int64_t tile = i >> 13;            // 8192 elements per tile
  const int rem = (int)(i & 8191);
  const int r = rem >> 6, pc = (rem >> 3) & 7, e = rem & 7;
  const int64_t mt = tile / KB, kb = tile % KB;
  *p = mt * 128 + r;
  *col = (int)(kb * 64 + ((pc ^ (r & 7)) << 3) + e);
}

__global__ void k_init_weights_tiled(bf16* out, int M, int K, int gu_ff, int rope_hd, uint64_t seed,
                                     int32_t tensor_id, float c) {
  const uint64_t key = seed ^ ((uint64_t)tensor_id << 40);
  const int KB = K / 64;
  const int64_t n = (int64_t)((M + 127) / 128) * 128 * K;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    int64_t p;
    int col;
    tiled_coords(i, KB, &p, &col);
    const int64_t lrow = tiled_logical_row(p, M, gu_ff, rope_hd);
    if (lrow < 0) {
      out[i] = __float2bfloat16_rn(0.f);
      continue;
    }
    const uint64_t u = splitmix64(key ^ (uint64_t)(lrow * K + col));
    const float v = __fsub_rn(__fmul_rn((float)(uint32_t)(u >> 40), 5.9604644775390625e-08f), 0.5f);
    out[i] = __float2bfloat16_rn(__fmul_rn(v, c));
  }
}

void launch_init_weights_tiled(bf16* out, int M, int K, int gu_ff, int rope_hd, uint64_t seed, int32_t tensor_id,
                               float sigma, cudaStream_t s) {
  const float c = (float)(2.0 * 1.7320508075688772 * (double)sigma);
  k_init_weights_tiled<<<148 * 64, 256, 0, s>>>(out, M, K, gu_ff, rope_hd, seed, tensor_id, c);
}

// row-major [M, K] -> tiled (zero-padded rows); used by the op-level GEMM entry points
__global__ void k_pack_tiled(const bf16* src, bf16* dst, int M, int K) {
  const int KB = K / 64;
  const int64_t n = (int64_t)((M + 127) / 128) * 128 * K;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    int64_t p;
    int col;
    tiled_coords(i, KB, &p, &col);
    dst[i] = p < M ? src[p * K + col] : __float2bfloat16_rn(0.f);
  }
}

void launch_pack_tiled(const bf16* src, bf16* dst, int M, int K, cudaStream_t s) {
  k_pack_tiled<<<148 * 16, 256, 0, s>>>(src, dst, M, K);
}

void launch_init_weights(bf16* out, int64_t n, uint64_t seed, int32_t tensor_id, float sigma,
                         cudaStream_t s) {
  const float c = (float)(2.0 * 1.7320508075688772 * (double)sigma);
  int blocks = (int)std::min<int64_t>((n + 255) / 256, 148 * 64);
  if (blocks < 1) blocks = 1;
  k_init_weights<<<blocks, 256, 0, s>>>(out, n, seed, tensor_id, c);
}

// ------------------------------------------------------------- block reduce
__device__ float block_sum(float v, float* red) {
  v = warp_sum(v);
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  __syncthreads();
  if (lane == 0) red[w] = v;
  __syncthreads();
  float t = 0.f;
  for (int i = 0; i < nw; ++i) t += red[i];
  return t;
}

// ---------------------------------------------------------------- embedding
// x[r] = emb[tok[r]] (fp32 residual), xb[r] = bf16(x[r]) (GEMM operand), ss[r][t] = sum of
// squares of x[r] over feature tile t (128 features) — the same un-normalised form the
// EPI_RESID epilogue leaves, so the first RMSNorm is applied by the QKV GEMM epilogue.
__global__ void k_embed(const int32_t* row_tok, int32_t row0, const bf16* emb, int d, int n_tiles, float* x,
                        bf16* xb, float* ss) {
  TraceScope tr(TK_EMBED);
  if (threadIdx.x == 0) pdl_trigger();
  pdl_wait();  // row_tok comes from the scheduler kernel
  tr.ready();
  const int r = blockIdx.x;
  const int tok = row_tok[row0 + r];
  const bf16* e = emb + (size_t)tok * d;
  float* xr = x + (size_t)r * d;
  bf16* hr = xb + (size_t)r * d;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  for (int t = warp; t < n_tiles; t += nw) {
    float sq = 0.f;
    for (int i = t * 128 + lane; i < min(d, t * 128 + 128); i += 32) {
      const bf16 b = e[i];
      const float v = __bfloat162float(b);
      xr[i] = v;
      hr[i] = b;
      sq += v * v;
    }
    sq = warp_sum(sq);
    if (lane == 0) ss[(size_t)r * n_tiles + t] = sq;
  }
}

// The same embedding for the first forward chunk of a scheduler round, launched right behind
// k_sched_pre BEFORE the host has read the plan: the row count comes from the device state
// the scheduler writes (min(*n_rows, fwd_rows)), rows in a grid-stride loop, so the launch
// does not depend on the plan and the embedding runs while the host completes the plan
// handshake and launches the layers (rt_step).
__global__ void k_embed_plan(const int32_t* row_tok, const int32_t* n_rows_dev, int fwd_rows, const bf16* emb,
                             int d, int n_tiles, float* x, bf16* xb, float* ss) {
  TraceScope tr(TK_EMBED);
  if (threadIdx.x == 0) pdl_trigger();
  pdl_wait();  // row_tok and the row count come from the scheduler kernel
  tr.ready();
  const int n = min(*n_rows_dev, fwd_rows);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  for (int r = blockIdx.x; r < n; r += gridDim.x) {
    const int tok = row_tok[r];
    const bf16* e = emb + (size_t)tok * d;
    float* xr = x + (size_t)r * d;
    bf16* hr = xb + (size_t)r * d;
    for (int t = warp; t < n_tiles; t += nw) {
      float sq = 0.f;
      for (int i = t * 128 + lane; i < min(d, t * 128 + 128); i += 32) {
        const bf16 b = e[i];
        const float v = __bfloat162float(b);
        xr[i] = v;
        hr[i] = b;
        sq += v * v;
      }
      sq = warp_sum(sq);
      if (lane == 0) ss[(size_t)r * n_tiles + t] = sq;
    }
  }
}

// RMSNorm scale of row r from the per-tile sums of squares (fixed order, shared with the
// GEMM epilogue's row scaling): rsqrt(sum_t ss[r][t] / d + 1e-5)
__device__ __forceinline__ float rms_inv(const float* ss, int n_tiles, int r, int d) {
  float t = 0.f;
  for (int i = 0; i < n_tiles; ++i) t += ss[(size_t)r * n_tiles + i];
  return rsqrtf(t / (float)d + 1e-5f);
}

// ------------------------------------------- gather logits rows + final RMSNorm
// hfin[s] = bf16(x[r] * rms_inv(r)), r = slot_row[s] - row0, for slots whose logits row
// lies in this chunk
__global__ void k_gather_norm(const int32_t* slot_row, int B, int row0, int n_rows, const float* x,
                              const float* ss, int n_tiles, int d, bf16* hfin) {
  TraceScope tr(TK_GATHER);
  if (threadIdx.x == 0) pdl_trigger();
  pdl_wait();
  tr.ready();
  const int s = blockIdx.x;
  if (s >= B) return;
  const int r = slot_row[s] - row0;
  if (r < 0 || r >= n_rows) return;
  __shared__ float inv;
  if (threadIdx.x == 0) inv = rms_inv(ss, n_tiles, r, d);
  __syncthreads();
  const float4* src = (const float4*)(x + (size_t)r * d);
  uint2* dst = (uint2*)(hfin + (size_t)s * d);
  for (int i = threadIdx.x; i < d / 4; i += blockDim.x) {
    const float4 v = src[i];
    dst[i] = make_uint2(pack_bf16x2(v.x * inv, v.y * inv), pack_bf16x2(v.z * inv, v.w * inv));
  }
}

// ------------------------------------------------------ residual split-K reduce
// Decode O / down projections in EPI_PART write their raw split-K partials part[s][n][m]; this
// kernel finishes them (oracle c1: x += o W_o^T, x += act W_d^T): x[n][m] += sum_s part (split
// order), the bf16 copy of x (the next projection's operand) and the per-128-feature sums of
// squares of the new x (the next RMSNorm, folded into its consumer).  CTA = (row n, 1024
// features), 256 threads x 4 features (float4); one warp = one 128-feature tile.
template <int S>
__global__ void __launch_bounds__(256) k_resid_reduce(const float* part, int ld_n, int M, float* x, bf16* xb,
                                                      float* ss) {
  TraceScope tr(TK_RESID);
  if (threadIdx.x == 0) pdl_trigger();
  pdl_wait();
  tr.ready();
  // CTA = (row n, 1024 features), thread = one float4 group; the split count is a template
  // parameter so the registers (and the one-wave occupancy of all CTAs) fit
  const int n = blockIdx.x;
  const int f = blockIdx.y * 1024 + threadIdx.x * 4;
  if (f >= M) return;  // (M % 128 == 0: whole warps)
  float4 w[S];
#pragma unroll
  for (int sp = 0; sp < S; ++sp) w[sp] = __ldcg(reinterpret_cast<const float4*>(part + ((size_t)sp * ld_n + n) * M + f));
  float4* xp = reinterpret_cast<float4*>(x + (size_t)n * M + f);
  const float4 xo = __ldcg(xp);
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
  for (int sp = 0; sp < S; ++sp) {
    acc.x += w[sp].x;
    acc.y += w[sp].y;
    acc.z += w[sp].z;
    acc.w += w[sp].w;
  }
  const float4 xn = make_float4(xo.x + acc.x, xo.y + acc.y, xo.z + acc.z, xo.w + acc.w);
  *xp = xn;
  *reinterpret_cast<uint2*>(xb + (size_t)n * M + f) = make_uint2(pack_bf16x2(xn.x, xn.y), pack_bf16x2(xn.z, xn.w));
  float q = ((xn.x * xn.x + xn.y * xn.y) + xn.z * xn.z) + xn.w * xn.w;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) q += __shfl_xor_sync(0xffffffffu, q, o);
  if ((threadIdx.x & 31) == 0) ss[(size_t)n * (M / 128) + f / 128] = q;
}
void launch_resid_reduce(const float* part, int S, int ld_n, int N, int M, float* x, bf16* xb, float* ss,
                         cudaStream_t s) {
  const dim3 grid(N, (M + 1023) / 1024), block(256);
  switch (S) {
#define RT_RR(k) \
  case k: launch_pdl(k_resid_reduce<k>, grid, block, 0, s, part, ld_n, M, x, xb, ss); break;
    RT_RR(1) RT_RR(2) RT_RR(3) RT_RR(4) RT_RR(5) RT_RR(6) RT_RR(7) RT_RR(8)
#undef RT_RR
    default: break;
  }
}

// ------------------------------------------------------ argmax final reduce
// part_val/part_idx [n_mtiles][N]; lowest index wins ties (c3)
__global__ void k_argmax_reduce(const float* part_val, const int32_t* part_idx, int n_mtiles, int N,
                                int32_t* tok) {
  TraceScope tr(TK_ARGMAX);
  if (threadIdx.x == 0) pdl_trigger();
  pdl_wait();
  tr.ready();
  const int n = blockIdx.x;
  float best = -INFINITY;
  int bi = INT_MAX;
  for (int t = threadIdx.x; t < n_mtiles; t += blockDim.x) {
    const float v = part_val[(size_t)t * N + n];
    const int i = part_idx[(size_t)t * N + n];
    if (v > best || (v == best && i < bi)) {
      best = v;
      bi = i;
    }
  }
  for (int o = 16; o > 0; o >>= 1) {
    const float ov = __shfl_xor_sync(0xffffffffu, best, o);
    const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
    if (ov > best || (ov == best && oi < bi)) {
      best = ov;
      bi = oi;
    }
  }
  __shared__ float sv[32];
  __shared__ int si[32];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) {
    sv[w] = best;
    si[w] = bi;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int j = 1; j < (int)(blockDim.x >> 5); ++j)
      if (sv[j] > best || (sv[j] == best && si[j] < bi)) {
        best = sv[j];
        bi = si[j];
      }
    tok[n] = bi;
  }
}

// --------------------------------------------------------- KV pool helpers
__global__ void k_kv_write(unsigned char* pool, const bf16* k, const bf16* v, const int32_t* slot, int nkv,
                           int hd) {
  const int r = blockIdx.x;
  const int sl = slot[r];
  const int page = sl / 16, off = sl % 16;
  for (int it = threadIdx.x; it < 2 * nkv * hd; it += blockDim.x) {
    const int kind = it / (nkv * hd);
    const int rem = it % (nkv * hd);
    const int h = rem / hd, d = rem % hd;
    const bf16 val = (kind == 0 ? k : v)[((size_t)r * nkv + h) * hd + d];
    unsigned char* blk = pool + (((size_t)page * nkv + h) * 2 + kind) * (size_t)(16 * hd * 2);
    *(bf16*)(blk + off * hd * 2 + (kv_swz_chunk(hd, off, d >> 3) << 4) + ((d & 7) << 1)) = val;
  }
}

// logical out [n_pages][2][nkv][16][hd]
__global__ void k_kv_read(const unsigned char* pool, bf16* out, int nkv, int hd) {
  const int page = blockIdx.x;
  for (int it = threadIdx.x; it < 2 * nkv * 16 * hd; it += blockDim.x) {
    int rem = it;
    const int d = rem % hd;
    rem /= hd;
    const int j = rem % 16;
    rem /= 16;
    const int h = rem % nkv;
    const int kind = rem / nkv;
    const unsigned char* blk = pool + (((size_t)page * nkv + h) * 2 + kind) * (size_t)(16 * hd * 2);
    out[(size_t)page * 2 * nkv * 16 * hd + it] =
        *(const bf16*)(blk + j * hd * 2 + (kv_swz_chunk(hd, j, d >> 3) << 4) + ((d & 7) << 1));
  }
}

// ------------------------------------------------------------- launchers
void launch_embed(const int32_t* row_tok, int row0, int n, const bf16* emb, int d, float* x, bf16* xb, float* ss,
                  cudaStream_t s) {
  launch_pdl(k_embed, dim3(n), dim3(256), 0, s, row_tok, row0, emb, d, (d + 127) / 128, x, xb, ss);
}
void launch_embed_plan(const int32_t* row_tok, const int32_t* n_rows_dev, int fwd_rows, const bf16* emb, int d,
                       float* x, bf16* xb, float* ss, cudaStream_t s) {
  launch_pdl(k_embed_plan, dim3(std::min(fwd_rows, 296)), dim3(256), 0, s, row_tok, n_rows_dev, fwd_rows, emb, d,
             (d + 127) / 128, x, xb, ss);
}
void launch_gather_norm(const int32_t* slot_row, int B, int row0, int n, const float* x, const float* ss, int d,
                        bf16* hfin, cudaStream_t s) {
  launch_pdl(k_gather_norm, dim3(B), dim3(128), 0, s, slot_row, B, row0, n, x, ss, (d + 127) / 128, d, hfin);
}
void launch_argmax_reduce(const float* pv, const int32_t* pi, int n_mtiles, int N, int32_t* tok,
                          cudaStream_t s) {
  launch_pdl(k_argmax_reduce, dim3(N), dim3(256), 0, s, pv, pi, n_mtiles, N, tok);
}
// KV eviction / restore (R-EVICT): entry i = (dir, task, device page, host
// page); block (i, layer) copies the page's [n_kv][K|V][16][hd] block of that layer between
// the device pool and the mapped pinned host pool ([host page][layer][block]), 16-byte
// vectors over PCIe (zero-copy: no staging buffer, no host involvement)
__global__ void k_kv_swap(const int4* swap, unsigned char* pool, int64_t pool_layer_bytes, unsigned char* host,
                          int64_t blk, int L) {
  const int4 w = swap[blockIdx.x];
  const int l = blockIdx.y;
  unsigned char* dev = pool + (size_t)l * pool_layer_bytes + (size_t)w.z * blk;
  unsigned char* hst = host + ((size_t)w.w * L + l) * blk;
  const uint4* src = reinterpret_cast<const uint4*>(w.x == 0 ? dev : hst);
  uint4* dst = reinterpret_cast<uint4*>(w.x == 0 ? hst : dev);
  for (int64_t j = threadIdx.x; j < blk / 16; j += blockDim.x) dst[j] = src[j];
}
void launch_kv_swap(const int4* swap, int n, void* pool, int64_t pool_layer_bytes, void* host, int64_t blk, int L,
                    cudaStream_t s) {
  if (n > 0)
    k_kv_swap<<<dim3(n, L), 256, 0, s>>>(swap, (unsigned char*)pool, pool_layer_bytes, (unsigned char*)host, blk,
                                         L);
}

void launch_kv_write(void* pool, const bf16* k, const bf16* v, const int32_t* slot, int n, int nkv, int hd,
                     cudaStream_t s) {
  k_kv_write<<<n, 256, 0, s>>>((unsigned char*)pool, k, v, slot, nkv, hd);
}
void launch_kv_read(const void* pool, bf16* out, int n_pages, int nkv, int hd, cudaStream_t s) {
  k_kv_read<<<n_pages, 256, 0, s>>>((const unsigned char*)pool, out, nkv, hd);
}

RT_TRACE_BINDER(trace_bind_model)

}  // namespace rt
