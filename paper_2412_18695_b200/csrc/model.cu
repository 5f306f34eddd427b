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

// ---------------------------------------------------- embedding + first norm
// x[r] = emb[tok[r]] (fp32), h[r] = bf16(rms(x[r]))
__global__ void k_embed_norm(const int32_t* row_tok, int32_t row0, const bf16* emb, int d, float* x,
                             bf16* h) {
  __shared__ float red[32];
  const int r = blockIdx.x;
  const int tok = row_tok[row0 + r];
  const bf16* e = emb + (size_t)tok * d;
  float* xr = x + (size_t)r * d;
  float ss = 0.f;
  for (int i = threadIdx.x; i < d; i += blockDim.x) {
    const float v = __bfloat162float(e[i]);
    xr[i] = v;
    ss += v * v;
  }
  const float tot = block_sum(ss, red);
  const float inv = rsqrtf(tot / (float)d + 1e-5f);
  bf16* hr = h + (size_t)r * d;
  for (int i = threadIdx.x; i < d; i += blockDim.x) hr[i] = __float2bfloat16_rn(xr[i] * inv);
}

// -------------------------------------------- residual add (+ next RMSNorm)
// x[r] += sum_s part[s][r][:];  h[r] = bf16(rms(x[r]))
__global__ void k_resid_norm(const float* part, int splits, int n_rows, int d, float* x, bf16* h) {
  __shared__ float red[32];
  const int r = blockIdx.x;
  float* xr = x + (size_t)r * d;
  float ss = 0.f;
  for (int i = threadIdx.x; i < d; i += blockDim.x) {
    float v = xr[i];
    for (int s = 0; s < splits; ++s) v += part[((size_t)s * n_rows + r) * d + i];
    xr[i] = v;
    ss += v * v;
  }
  const float tot = block_sum(ss, red);
  const float inv = rsqrtf(tot / (float)d + 1e-5f);
  bf16* hr = h + (size_t)r * d;
  for (int i = threadIdx.x; i < d; i += blockDim.x) hr[i] = __float2bfloat16_rn(xr[i] * inv);
}

// ------------------------------------------------------------ SwiGLU product
// a[r][j] = bf16(silu(g) * u), g = gu[j], u = gu[ff + j]
__global__ void k_swiglu(const float* part, int splits, int n_rows, int ff, bf16* act) {
  const int r = blockIdx.y;
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < ff; j += gridDim.x * blockDim.x) {
    float g = 0.f, u = 0.f;
    for (int s = 0; s < splits; ++s) {
      const float* p = part + ((size_t)s * n_rows + r) * (2 * ff);
      g += p[j];
      u += p[ff + j];
    }
    const float sg = g / (1.f + __expf(-g));
    act[(size_t)r * ff + j] = __float2bfloat16_rn(sg * u);
  }
}

// ------------------------------------------- QKV epilogue: RoPE + KV append
// part: [splits][n_rows][(nq + 2 nkv) hd]; q_out bf16 [n_rows][nq][hd];
// K/V written (bf16) into the swizzled pool of this layer at the row's position.
__global__ void k_qkv_epilogue(QkvEpiArgs a) {
  const int r = blockIdx.x;
  const int hd = a.hd, half = hd / 2;
  const int row = a.row0 + r;
  const int task = a.row_task[row];
  const int pos = a.row_pos[row];
  const int n_pairs = (a.nq + 2 * a.nkv) * half;
  const int qkv_dim = (a.nq + 2 * a.nkv) * hd;
  const int page = a.page_table[(size_t)task * a.pt_stride + pos / 16];
  const int off = pos % 16;
  const float* cs = a.rope_cos + (size_t)pos * half;
  const float* sn = a.rope_sin + (size_t)pos * half;
  for (int it = threadIdx.x; it < n_pairs; it += blockDim.x) {
    const int head = it / half, i = it % half;
    const int col = head * hd + i;
    float x1 = 0.f, x2 = 0.f;
    for (int s = 0; s < a.splits; ++s) {
      const float* p = a.part + ((size_t)s * a.n_rows + r) * qkv_dim;
      x1 += p[col];
      x2 += p[col + half];
    }
    if (head < a.nq + a.nkv) {  // q or k: rotate-half RoPE (theta 500000)
      const float c = cs[i], s_ = sn[i];
      const float y1 = x1 * c - x2 * s_;
      const float y2 = x2 * c + x1 * s_;
      x1 = y1;
      x2 = y2;
    }
    const bf16 b1 = __float2bfloat16_rn(x1), b2 = __float2bfloat16_rn(x2);
    if (head < a.nq) {
      bf16* q = a.q_out + ((size_t)r * a.nq + head) * hd;
      q[i] = b1;
      q[i + half] = b2;
      if (a.q_cap) {
        float* qc = a.q_cap + ((size_t)row * a.nq + head) * hd;
        qc[i] = __bfloat162float(b1);
        qc[i + half] = __bfloat162float(b2);
      }
    } else {
      const int kind = head < a.nq + a.nkv ? 0 : 1;
      const int kvh = kind == 0 ? head - a.nq : head - a.nq - a.nkv;
      unsigned char* blk = (unsigned char*)a.pool +
                           (((size_t)page * a.nkv + kvh) * 2 + kind) * (size_t)(16 * hd * 2);
      const int c1 = i >> 3, c2 = (i + half) >> 3;
      *(bf16*)(blk + off * hd * 2 + (kv_swz_chunk(hd, off, c1) << 4) + ((i & 7) << 1)) = b1;
      *(bf16*)(blk + off * hd * 2 + (kv_swz_chunk(hd, off, c2) << 4) + (((i + half) & 7) << 1)) = b2;
    }
  }
}

// -------------------------------------------------- gather logits rows
// hfin[s] = h[slot_row[s] - row0] for slots whose logits row lies in this chunk
__global__ void k_gather_rows(const int32_t* slot_row, int B, int row0, int n_rows, const bf16* h, int d,
                              bf16* hfin) {
  const int s = blockIdx.x;
  if (s >= B) return;
  const int r = slot_row[s] - row0;
  if (r < 0 || r >= n_rows) return;
  const uint4* src = (const uint4*)(h + (size_t)r * d);
  uint4* dst = (uint4*)(hfin + (size_t)s * d);
  for (int i = threadIdx.x; i < d / 8; i += blockDim.x) dst[i] = src[i];
}

// ------------------------------------------------------ argmax final reduce
// part_val/part_idx [n_mtiles][N]; lowest index wins ties (c3)
__global__ void k_argmax_reduce(const float* part_val, const int32_t* part_idx, int n_mtiles, int N,
                                int32_t* tok) {
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
void launch_embed_norm(const int32_t* row_tok, int row0, int n, const bf16* emb, int d, float* x, bf16* h,
                       cudaStream_t s) {
  k_embed_norm<<<n, 256, 0, s>>>(row_tok, row0, emb, d, x, h);
}
void launch_resid_norm(const float* part, int splits, int n, int d, float* x, bf16* h, cudaStream_t s) {
  k_resid_norm<<<n, 256, 0, s>>>(part, splits, n, d, x, h);
}
void launch_swiglu(const float* part, int splits, int n, int ff, bf16* act, cudaStream_t s) {
  dim3 g((ff + 255) / 256 < 8 ? (ff + 255) / 256 : 8, n);
  k_swiglu<<<g, 256, 0, s>>>(part, splits, n, ff, act);
}
void launch_qkv_epilogue(const QkvEpiArgs& a, cudaStream_t s) { k_qkv_epilogue<<<a.n_rows, 256, 0, s>>>(a); }
void launch_gather_rows(const int32_t* slot_row, int B, int row0, int n, const bf16* h, int d, bf16* hfin,
                        cudaStream_t s) {
  k_gather_rows<<<B, 128, 0, s>>>(slot_row, B, row0, n, h, d, hfin);
}
void launch_argmax_reduce(const float* pv, const int32_t* pi, int n_mtiles, int N, int32_t* tok,
                          cudaStream_t s) {
  k_argmax_reduce<<<N, 256, 0, s>>>(pv, pi, n_mtiles, N, tok);
}
void launch_kv_write(void* pool, const bf16* k, const bf16* v, const int32_t* slot, int n, int nkv, int hd,
                     cudaStream_t s) {
  k_kv_write<<<n, 256, 0, s>>>((unsigned char*)pool, k, v, slot, nkv, hd);
}
void launch_kv_read(const void* pool, bf16* out, int n_pages, int nkv, int hd, cudaStream_t s) {
  k_kv_read<<<n_pages, 256, 0, s>>>((const unsigned char*)pool, out, nkv, hd);
}

}  // namespace rt
