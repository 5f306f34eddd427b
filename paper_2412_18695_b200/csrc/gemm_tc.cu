// gemm_tc.cu — dense projections on 5th-gen tensor cores with fused epilogues
// (SURVEY §8(a) a6, a8).
//
//   D[m, n] = sum_k W[m, k] * X[n, k]        (bf16 x bf16 -> fp32 in TMEM)
//
// Decode projections are skinny (N = running batch): the weight matrix goes in the
// UMMA M slot (128 rows per tile) and the batch in N (32..256), so the weights
// stream through HBM once per step (HBM-bound for N <~ 210).
//
// Split-K across a THREAD-BLOCK CLUSTER (k_gemm_tc, <= 128 rows): the S CTAs of a
// cluster (grid.x = S, up to 16 with the non-portable opt-in) stream disjoint K ranges
// of the same 128 x BN tile into their own TMEM accumulators; each then parks its fp32
// partial in its own shared memory and, after one cluster barrier, PUSHES the column
// slice every peer owns into that peer's receive slot (cp.async.bulk.shared::cluster,
// mbarrier complete_tx); CTA r sums the S slices of its columns [r BN / S, (r+1) BN / S)
// in fixed rank order (deterministic) and applies the fused epilogue to them.  No
// global workspace, no atomics, the reduction runs on all S SMs in parallel.  S comes
// from gemm_choose_splits: the largest S <= 8 with S x tiles <= 256 co-resident CTAs
// (128 for 192/256-wide tiles) and >= 4 k-blocks per split — at the 8B decode shapes
// QKV 48 tiles x 5, O / down 32 x 8, gate-up / lm_head (>= 148 tiles) unsplit.  EPI_PART
// (decode QKV / O / down) skips the exchange: every split writes its
// raw fp32 partial and the consumer (k_attn's QKV fold, k_resid_reduce) sums them.
// CTA roles (192 threads):
//   warp 0 lane 0 : TMA producer — weights are stored in HBM as UMMA-ready 16 KiB
//                   SW128 tiles, so each k-block of W is ONE
//                   cp.async.bulk of a contiguous range (a CTA streams sequential
//                   HBM); X [BN x 64] tiles come by cp.async.bulk.tensor.2d; the
//                   weight tiles of the first stages are requested BEFORE
//                   griddepcontrol.wait (programmatic dependent launch), so weight
//                   streaming overlaps the previous kernel's tail;
//   warp 1        : TMEM allocator; lane 0 issues tcgen05.mma.cta_group::1.kind::f16
//                   (M=128, N=BN, K=16), tcgen05.commit frees stages / signals the epilogue;
//   warps 2..5    : epilogue — tcgen05.ld.32x32b.x16 (lane quarter = warp % 4) parks
//                   the accumulator in shared memory; split-K partials are exchanged
//                   inside the cluster (DSMEM bulk push, fixed-order sum); then a compact
//                   4-column loop applies the fused op of oracle c1 (the RMSNorm of the
//                   input folded in as a per-column scale, g.rs_ss):
//        EPI_STORE  fp32 out[n][m]
//        EPI_ARGMAX lm_head: per-tile (max, lowest index) + optional logits
//        EPI_QKV    RoPE (rotate-half, theta 5e5) on q/k, bf16 q out, bf16 K/V
//                   appended into the swizzled KV page of (row task, position); the
//                   rotate-half partners are adjacent weight rows (lane shuffle)
//        EPI_RESID  x[n][m] += D (fp32 residual stream), bf16 copy for the next GEMM,
//                   per-tile sum of squares of the new x for the next RMSNorm
//        EPI_SWIGLU gate / up rows adjacent per feature: act = bf16(silu(g) u)
#include <cuda.h>
#include <cudaTypedefs.h>
#include "common.cuh"
#include "model.h"
#include <map>
#include <mutex>
#include <utility>

namespace rt {

constexpr int kGemmThreads = 192;
constexpr int kDecThreads = 320;  // CTA-pair kernels: producer, MMA, 2 x 4 epilogue warps
constexpr int kBK = 64;  // one 128-byte swizzle atom of bf16 along K

template <int BN>
struct GemmCfg {
  static constexpr int A_BYTES = 128 * kBK * 2;    // 16 KB
  static constexpr int B_BYTES = BN * kBK * 2;
  static constexpr int STAGE = A_BYTES + B_BYTES;
  static constexpr int STAGES = BN <= 64 ? 4 : (BN == 128 ? 3 : (BN == 256 ? 4 : 5));
  static constexpr int CTAS_PER_SM = BN <= 128 ? 2 : 1;
  static constexpr int TMEM_COLS = BN <= 32 ? 32 : BN <= 64 ? 64 : BN <= 128 ? 128 : 256;  // power of 2
  static constexpr int META = 3 * BN * 4;                       // per-column pos / page / rms scale
  static constexpr int RED = 2 * 4 * BN * 4;                    // per-warp column partials (val, idx)
  static constexpr int XP = 16 * 128 * 4;                       // prefetched epilogue inputs
  static constexpr int SMEM = 1024 + STAGES * STAGE + 512 + META + RED + XP;
  static_assert(BN * 128 * 4 <= STAGES * STAGE, "partial tile must fit in the ring");
  static_assert(BN > 128 || SMEM + 1024 <= 233472 / 2, "two CTAs per SM");
  // push reduction: partial tile + S receive slots of ceil(BN/S) columns (<= BN + 16
  // columns for S <= 16 ... checked per launch) fit in the ring
  static constexpr bool PUSH = (2 * BN + 16) * 128 * 4 <= STAGES * STAGE;
};

// ------------------------------------------------------------------ PTX
__device__ __forceinline__ void tma_load_2d(void* dst, const void* tmap, int c0, int c1, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], "
      "[%4];" ::"r"(smem_u32(dst)),
      "l"(tmap), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void prefetch_tmap(const void* tmap) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(tmap) : "memory");
}
// UMMA shared-memory descriptor, K-major SWIZZLE_128B (CUTLASS UMMA::SmemDescriptor):
// start>>4 [0,14) | LBO>>4 [16,30) | SBO>>4 [32,46) | version 1 [46,48) | layout 2 [61,64)
__device__ __forceinline__ uint64_t umma_desc_sw128(uint32_t saddr) {
  uint64_t d = (uint64_t)((saddr & 0x3FFFF) >> 4);
  d |= (uint64_t)1 << 16;              // LBO (unused for swizzled K-major)
  d |= (uint64_t)(1024 >> 4) << 32;    // SBO: 8 rows x 128 B
  d |= (uint64_t)1 << 46;              // version (sm_100)
  d |= (uint64_t)2 << 61;              // SWIZZLE_128B
  return d;
}
// instruction descriptor kind::f16: D f32, A/B bf16, K-major, N>>3 at [17,23), M>>4 at [24,29)
__host__ __device__ constexpr uint32_t umma_idesc(int M, int N) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}
__device__ __forceinline__ void umma_f16(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                         uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}
__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float* v) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, "
      "[%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]),
        "=r"(r[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}
// named barrier of one 128-thread epilogue group (id 1; the decode pair kernel's second
// group uses id 2)
__device__ __forceinline__ void epi_bar(int id = 1) { asm volatile("bar.sync %0, 128;" ::"r"(id) : "memory"); }
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
// address of the same shared-memory location in CTA `rank` of the cluster
__device__ __forceinline__ uint32_t dsmem_addr(uint32_t local, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(local), "r"(rank));
  return r;
}
__device__ __forceinline__ float ld_dsmem(uint32_t addr) {
  float v;
  asm volatile("ld.shared::cluster.f32 %0, [%1];" : "=f"(v) : "r"(addr) : "memory");
  return v;
}

struct EpiSmem {
  int* pos;      // [BN] KV position of each column's row (EPI_QKV)
  int* page;     // [BN] KV page of each column's row (EPI_QKV)
  float* inv;    // [BN] per-column RMSNorm scale (g.rs_ss)
  int bn;
  float* redv;   // [4][BN] per-warp column partials (EPI_RESID sum of squares, EPI_ARGMAX max)
  int* redi;     // [4][BN] per-warp argmax index
  int xp_sin;    // offset (floats) of the sin table in xp (EPI_QKV)
  float* xp;     // [16][128] epilogue inputs prefetched during the mainloop (EPI_RESID x;
                 //  EPI_QKV cos [16][64] then sin [16][64])
  long long* mark;  // clock64 phase marks (trace), written by thread et == 0
  bf16* stg = nullptr;  // nullable: EPI_QKV staging [2][16][128] bf16 (whole head rows, 16-byte stores)
  int bar = 1;          // named barrier of this epilogue group (128 threads)
};
#define EPI_MARK(i) \
  if (et == 0 && sm.mark) sm.mark[i] = clock64()

// Reductions of 4 columns across the 32 lanes at once (reduce-scatter: 6 shuffles instead
// of 4 x 5): the result for column j = (lane >> 3) & 3 ends on lanes with lane & 7 == 0.
__device__ __forceinline__ float warp_sum4(const float (&v)[4], int lane) {
  const bool hi16 = lane & 16, hi8 = lane & 8;
  float a0 = hi16 ? v[2] : v[0], a1 = hi16 ? v[3] : v[1];
  const float b0 = hi16 ? v[0] : v[2], b1 = hi16 ? v[1] : v[3];
  a0 += __shfl_xor_sync(0xffffffffu, b0, 16);
  a1 += __shfl_xor_sync(0xffffffffu, b1, 16);
  float c = hi8 ? a1 : a0;
  const float d = hi8 ? a0 : a1;
  c += __shfl_xor_sync(0xffffffffu, d, 8);
  c += __shfl_xor_sync(0xffffffffu, c, 4);
  c += __shfl_xor_sync(0xffffffffu, c, 2);
  c += __shfl_xor_sync(0xffffffffu, c, 1);
  return c;
}
__device__ __forceinline__ void amax_merge(float& bv, int& bi, float ov, int oi) {
  const bool t = ov > bv || (ov == bv && oi < bi);  // selects, no branch
  bv = t ? ov : bv;
  bi = t ? oi : bi;
}
// (max, lowest index on ties) of 4 columns, same lane mapping as warp_sum4
__device__ __forceinline__ void warp_argmax4(const float (&v)[4], const int (&ix)[4], int lane, float& rv, int& ri) {
  const bool hi16 = lane & 16, hi8 = lane & 8;
  float a0 = hi16 ? v[2] : v[0], a1 = hi16 ? v[3] : v[1];
  int i0 = hi16 ? ix[2] : ix[0], i1 = hi16 ? ix[3] : ix[1];
  const float b0 = hi16 ? v[0] : v[2], b1 = hi16 ? v[1] : v[3];
  const int j0 = hi16 ? ix[0] : ix[2], j1 = hi16 ? ix[1] : ix[3];
  amax_merge(a0, i0, __shfl_xor_sync(0xffffffffu, b0, 16), __shfl_xor_sync(0xffffffffu, j0, 16));
  amax_merge(a1, i1, __shfl_xor_sync(0xffffffffu, b1, 16), __shfl_xor_sync(0xffffffffu, j1, 16));
  rv = hi8 ? a1 : a0;
  ri = hi8 ? i1 : i0;
  const float d = hi8 ? a0 : a1;
  const int di = hi8 ? i0 : i1;
  amax_merge(rv, ri, __shfl_xor_sync(0xffffffffu, d, 8), __shfl_xor_sync(0xffffffffu, di, 8));
#pragma unroll
  for (int o = 4; o > 0; o >>= 1)
    amax_merge(rv, ri, __shfl_xor_sync(0xffffffffu, rv, o), __shfl_xor_sync(0xffffffffu, ri, o));
}

// Where the finished tile's value (column c, row r) comes from: this CTA's parked partial
// P [BN][128] (S = 1), or the S split-K partials summed in fixed rank order from the local
// receive slots (push) or from the peers' P over DSMEM (pull).
struct TileSrc {
  const float* P;
  const float* R;
  uint32_t pl;  // smem address of P (pull)
  int S, rank, slot_cols, cb, kind;  // kind 0 local, 1 push, 2 pull
};
// Epilogue chunk: 16 columns per iteration.  The loop is latency-bound (4 epilogue warps,
// one per SM sub-partition, nothing else to hide behind), so every load of a chunk is
// issued before any of its math and the 4-column reductions of a chunk are independent
// chains (measured: 4 columns per iteration ran at ~500 cycles per iteration).
constexpr int kEpiCh = 16;
__device__ __forceinline__ float lds_f32(uint32_t a) {
  float v;
  asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(a));
  return v;
}
// v[k] = value of columns c0 + k (k < 16, columns >= ce read as 0) at row r (explicit
// shared-window loads: P / R are shared memory)
__device__ __forceinline__ void tile_vals16(const TileSrc& t, int c0, int ce, int r, float (&v)[kEpiCh]) {
  if (t.kind == 0) {
    const uint32_t base = smem_u32(t.P) + (uint32_t)((c0 * 128 + r) * 4);
#pragma unroll
    for (int k = 0; k < kEpiCh; ++k) v[k] = (c0 + k < ce) ? lds_f32(base + k * 512) : 0.f;
    return;
  }
#pragma unroll
  for (int k = 0; k < kEpiCh; ++k) v[k] = 0.f;
#pragma unroll 1
  for (int rk = 0; rk < t.S; ++rk) {
    float w[kEpiCh];
    if (t.kind == 1) {
      const float* src = rk == t.rank ? t.P + (size_t)c0 * 128 : t.R + ((size_t)rk * t.slot_cols + (c0 - t.cb)) * 128;
      const uint32_t base = smem_u32(src) + (uint32_t)(r * 4);
#pragma unroll
      for (int k = 0; k < kEpiCh; ++k) w[k] = (c0 + k < ce) ? lds_f32(base + k * 512) : 0.f;
    } else {
      const uint32_t base = dsmem_addr(t.pl, (uint32_t)rk) + (uint32_t)((c0 * 128 + r) * 4);
#pragma unroll
      for (int k = 0; k < kEpiCh; ++k) w[k] = (c0 + k < ce) ? ld_dsmem(base + k * 512) : 0.f;
    }
#pragma unroll
    for (int k = 0; k < kEpiCh; ++k) v[k] += w[k];
  }
}

// ------------------------------------------------------------ fused epilogue ops
// The finished columns [cb, ce) of this CTA, kEpiCh per iteration of a non-unrolled loop
// (the epilogue runs once per CTA; one chunk body keeps the code small), inlined at ONE
// call site (a non-inlined call would pass the kernel parameters through local memory).
// All 128 epilogue threads call it (named barrier at the end).
template <int MODE>
__device__ __forceinline__ void epilogue(const GemmArgs& g, const EpiSmem& sm, const TileSrc& ts, int m_tile,
                                      int n0, int cb, int ce, int et, bool pre) {
  constexpr int CH = kEpiCh;
  const int m0 = m_tile * 128;
  const int m = m0 + et;
  const int lane = et & 31, wq = et >> 5;
  const int NL = min(g.N - n0, ce);  // columns >= NL are out of range
  // The pairwise ops read the partner row from the adjacent TMEM lane (et ^ 1; the weight
  // rows are laid out pairwise, tiled_logical_row in model.cu) with one shuffle.
  bool active = m < g.M;
  if constexpr (MODE == EPI_SWIGLU) active = m_tile * 64 + (et >> 1) < g.ff;
  // global inputs of a chunk (EPI_RESID: residual x; EPI_QKV: cos / sin of the rotation),
  // from the mainloop-time prefetch (pre) or software-pipelined one chunk ahead so a long
  // column loop (prefill rows) does not pay a memory round trip per chunk
  constexpr bool HAS_IN = MODE == EPI_RESID || MODE == EPI_QKV;
  const int qi = (MODE == EPI_QKV) ? (et % g.qkv.hd) >> 1 : 0;
  const bool qrope = (MODE == EPI_QKV) && (m / g.qkv.hd) < g.qkv.nq + g.qkv.nkv;
  auto load_in = [&](int c, float (&ia)[CH], float (&ib)[CH]) {
    // predicated loads (no per-column branches, so all 16 are in flight at once)
#pragma unroll
    for (int k = 0; k < CH; ++k) {
      const bool ok = active && c + k < NL;
      if constexpr (MODE == EPI_RESID) {
        ia[k] = !ok ? 0.f : pre ? sm.xp[(c - cb + k) * 128 + et] : g.x[(size_t)(n0 + c + k) * g.M + m];
        ib[k] = 0.f;
      } else if constexpr (MODE == EPI_QKV) {
        const bool okr = ok && qrope;
        const int half = g.qkv.hd >> 1;
        if (pre) {
          ia[k] = okr ? sm.xp[(c - cb + k) * 64 + qi] : 0.f;
          ib[k] = okr ? sm.xp[sm.xp_sin + (c - cb + k) * 64 + qi] : 0.f;
        } else {
          const int pos = okr ? sm.pos[c + k] : 0;
          ia[k] = okr ? g.qkv.cos[(size_t)pos * half + qi] : 0.f;
          ib[k] = okr ? g.qkv.sin[(size_t)pos * half + qi] : 0.f;
        }
      } else {
        ia[k] = ib[k] = 0.f;
      }
    }
  };
  float in_a[CH], in_b[CH];
  if constexpr (HAS_IN) load_in(cb, in_a, in_b);
#pragma unroll 1
  for (int c0 = cb; c0 < ce; c0 += CH) {
    float ca[CH], cbv[CH];
    if constexpr (HAS_IN) {
#pragma unroll
      for (int k = 0; k < CH; ++k) {
        ca[k] = in_a[k];
        cbv[k] = in_b[k];
      }
      if (c0 + CH < ce) load_in(c0 + CH, in_a, in_b);
    }
    float v[CH], u[CH];
    tile_vals16(ts, c0, ce, et, v);
    if (et == 0 && c0 == cb && sm.mark) {  // trace: partial sums loaded (data-dependent mark)
      const long long t = clock64() + (v[0] == 1.2345e-30f ? 1 : 0);
      sm.mark[4] = t;
      sm.mark[5] = t;
    }
    if (g.rs_ss) {
      const uint32_t ib = smem_u32(sm.inv + c0);
#pragma unroll
      for (int k = 0; k < CH; ++k) v[k] *= (c0 + k < NL) ? lds_f32(ib + 4 * k) : 0.f;
    }
    if (MODE == EPI_SWIGLU || MODE == EPI_QKV)
#pragma unroll
      for (int k = 0; k < CH; ++k) u[k] = __shfl_xor_sync(0xffffffffu, v[k], 1);
    if constexpr (MODE == EPI_STORE) {
      if (active)
#pragma unroll
        for (int k = 0; k < CH; ++k)
          if (c0 + k < NL) g.out[(size_t)(n0 + c0 + k) * g.M + m] = v[k];
    } else if constexpr (MODE == EPI_RESID) {
      // math first for all columns (no branches: independent chains interleave), then
      // the guarded stores
      float sq[CH], xn[CH];
#pragma unroll
      for (int k = 0; k < CH; ++k) {
        xn[k] = (active && c0 + k < NL) ? ca[k] + v[k] : 0.f;
        sq[k] = xn[k] * xn[k];
      }
      if (active)
#pragma unroll
        for (int k = 0; k < CH; ++k)
          if (c0 + k < NL) g.x[(size_t)(n0 + c0 + k) * g.M + m] = xn[k];
      if (active && g.xb)
#pragma unroll
        for (int k = 0; k < CH; ++k)
          if (c0 + k < NL) g.xb[(size_t)(n0 + c0 + k) * g.M + m] = __float2bfloat16_rn(xn[k]);
#pragma unroll
      for (int j = 0; j < CH / 4; ++j) {
        const float q4[4] = {sq[4 * j], sq[4 * j + 1], sq[4 * j + 2], sq[4 * j + 3]};
        const float t = warp_sum4(q4, lane);  // column c0 + 4j + ((lane >> 3) & 3) on lanes 8i
        const int c = c0 + 4 * j + ((lane >> 3) & 3);
        if ((lane & 7) == 0 && c < ce) sm.redv[wq * sm.bn + c] = t;
      }
    } else if constexpr (MODE == EPI_SWIGLU) {
      // even lane: gate row, odd lane: up row of feature jf; the even lane writes the first
      // two columns of each group of 4 and the odd lane the last two.  Math for the 8
      // columns of this lane first (selects, no branches), then the guarded stores.
      const bool odd = et & 1;
      const int jf = m_tile * 64 + (et >> 1);
      float h[CH / 2];
#pragma unroll
      for (int j = 0; j < CH / 2; ++j) {
        const int ka = 4 * (j >> 1) + (j & 1), kb = ka + 2;
        const float gv = odd ? u[kb] : v[ka], uv = odd ? v[kb] : u[ka];
        h[j] = __fdividef(gv, 1.f + __expf(-gv)) * uv;
      }
      if (active)
#pragma unroll
        for (int j = 0; j < CH / 2; ++j) {
          const int c = c0 + 4 * (j >> 1) + (j & 1) + (odd ? 2 : 0);
          if (c < NL) g.act[(size_t)(n0 + c) * g.ff + jf] = __float2bfloat16_rn(h[j]);
        }
    } else if constexpr (MODE == EPI_QKV) {
      // row 2i of a head = dim i, row 2i + 1 = dim i + hd/2 (rotate-half partners); every
      // lane produces its own dim: y_i = x_i cos - x_{i+h} sin, y_{i+h} = x_{i+h} cos + x_i sin
      const QkvFuse& q = g.qkv;
      const int hd = q.hd, half = hd >> 1;
      const int r = et % hd, i = r >> 1;
      const bool odd = r & 1;
      const int dim = odd ? i + half : i;
      const int head = m / hd;
      const bool rope = head < q.nq + q.nkv;
      bf16 yb[CH];  // math first (no branches), then the guarded stores
#pragma unroll
      for (int k = 0; k < CH; ++k) {
        const float y = rope ? (odd ? v[k] * ca[k] + u[k] * cbv[k] : v[k] * ca[k] - u[k] * cbv[k]) : v[k];
        yb[k] = __float2bfloat16_rn(y);
      }
      if (sm.stg && hd == 128 && !q.q_cap) {
        // staged: the 128 rows of this m-tile are one head (CTA-uniform q / k / v); the chunk's
        // 16 head rows (256 B each) go out as 16-byte stores, 2 per thread (2-byte scattered
        // stores made this loop store-bound at 256 rows: ~8 us for 96 columns)
        bf16* st = sm.stg + (((c0 - cb) / CH) & 1) * (CH * 128);
#pragma unroll
        for (int k = 0; k < CH; ++k) st[k * 128 + dim] = yb[k];
        epi_bar(sm.bar);
        if (active) {
          const int kind = head < q.nq ? 2 : (rope ? 0 : 1);
          const int kvh = kind == 0 ? head - q.nq : head - q.nq - q.nkv;
#pragma unroll
          for (int w = 0; w < 2; ++w) {
            const int item = et + 128 * w, k = item >> 4, cc = item & 15;
            const int c = c0 + k;
            if (c < NL) {
              const uint4 val = *reinterpret_cast<const uint4*>(st + k * 128 + cc * 8);
              unsigned char* dst;
              if (kind == 2) {
                dst = (unsigned char*)(q.q_out + ((size_t)(n0 + c) * q.nq + head) * 128) + cc * 16;
              } else {
                const int pos = sm.pos[c], pg = sm.page[c], off = pos & 15;
                dst = (unsigned char*)q.pool + (((size_t)pg * q.nkv + kvh) * 2 + kind) * (size_t)(16 * 128 * 2) +
                      off * 256 + (kv_swz_chunk(128, off, cc) << 4);
              }
              *reinterpret_cast<uint4*>(dst) = val;
            }
          }
        }
      } else if (active) {
        if (head < q.nq) {  // warp-uniform (a head is 128 rows)
#pragma unroll
          for (int k = 0; k < CH; ++k)
            if (c0 + k < NL) q.q_out[((size_t)(n0 + c0 + k) * q.nq + head) * hd + dim] = yb[k];
          if (q.q_cap)
#pragma unroll
            for (int k = 0; k < CH; ++k)
              if (c0 + k < NL)
                q.q_cap[((size_t)(q.row0 + n0 + c0 + k) * q.nq + head) * hd + dim] = __bfloat162float(yb[k]);
        } else {
          // KV append into the swizzled page of (row task, position): addresses of all
          // columns first (predicated shared loads), then the stores
          const int kind = rope ? 0 : 1;
          const int kvh = kind == 0 ? head - q.nq : head - q.nq - q.nkv;
          unsigned char* dst[CH];
#pragma unroll
          for (int k = 0; k < CH; ++k) {
            const bool ok = c0 + k < NL;
            const int pos = ok ? sm.pos[c0 + k] : 0, pg = ok ? sm.page[c0 + k] : 0;
            const int off = pos & 15;
            dst[k] = (unsigned char*)q.pool + (((size_t)pg * q.nkv + kvh) * 2 + kind) * (size_t)(16 * hd * 2) +
                     off * hd * 2 + (kv_swz_chunk(hd, off, dim >> 3) << 4) + ((dim & 7) << 1);
          }
#pragma unroll
          for (int k = 0; k < CH; ++k)
            if (c0 + k < NL) *(bf16*)dst[k] = yb[k];
        }
      }
    } else if constexpr (MODE == EPI_ARGMAX) {
      if (g.out && active)  // logits (parity mode only)
#pragma unroll
        for (int k = 0; k < CH; ++k)
          if (c0 + k < NL) g.out[(size_t)(n0 + c0 + k) * g.M + m] = v[k];
#pragma unroll
      for (int j = 0; j < CH / 4; ++j) {
        float bv[4];
        int bi[4];
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) {  // greedy: max over the tile's rows, lowest index on ties
          const int k = 4 * j + kk;
          const bool ok = active && c0 + k < NL;
          bv[kk] = ok ? v[k] : -INFINITY;
          bi[kk] = ok ? m : INT_MAX;
        }
        float rv;
        int ri;
        warp_argmax4(bv, bi, lane, rv, ri);  // column c0 + 4j + ((lane >> 3) & 3) on lanes 8i
        const int c = c0 + 4 * j + ((lane >> 3) & 3);
        if ((lane & 7) == 0 && c < ce) {
          sm.redv[wq * sm.bn + c] = rv;
          sm.redi[wq * sm.bn + c] = ri;
        }
      }
    }
  }
  EPI_MARK(6);
  if constexpr (MODE == EPI_RESID || MODE == EPI_ARGMAX) {
    epi_bar(sm.bar);
    for (int c = cb + et; c < NL; c += 128) {  // fixed order over the 4 row quarters
      if constexpr (MODE == EPI_RESID) {
        const float t = ((sm.redv[c] + sm.redv[sm.bn + c]) + sm.redv[2 * sm.bn + c]) + sm.redv[3 * sm.bn + c];
        g.ss[(size_t)(n0 + c) * ((g.M + 127) / 128) + m_tile] = t;
      } else {
        float bv = sm.redv[c];
        int bi = sm.redi[c];
        for (int w = 1; w < 4; ++w) {
          const float ov = sm.redv[w * sm.bn + c];
          const int oi = sm.redi[w * sm.bn + c];
          if (ov > bv || (ov == bv && oi < bi)) {
            bv = ov;
            bi = oi;
          }
        }
        g.part_val[(size_t)m_tile * g.N + n0 + c] = bv;
        g.part_idx[(size_t)m_tile * g.N + n0 + c] = bi;
      }
    }
  }
  EPI_MARK(7);
}

// Per-column metadata of columns [cb, ce) for the 128 epilogue threads: KV position /
// page of the row (EPI_QKV) and the RMSNorm scale of the row (g.rs_ss; summation order
// of the per-tile sums fixed, t = 0 .. rs_tiles - 1).  Then, when the CTA finishes at most
// 16 columns, its epilogue's global inputs are prefetched into sm.xp while the mainloop
// runs (returns true).
template <int MODE>
__device__ __forceinline__ bool column_meta(const GemmArgs& g, const EpiSmem& sm, int m_tile, int n0, int cb, int ce,
                                         int et, bool allow_pre = true) {
  if (MODE != EPI_QKV && MODE != EPI_RESID && !g.rs_ss) return false;
  for (int cc = cb + et; cc < ce; cc += 128) {
    const int n = n0 + cc;
    if (n >= g.N) {
      sm.inv[cc] = 0.f;
      continue;
    }
    if (MODE == EPI_QKV) {
      const int row = g.qkv.row0 + n;
      const int pos = g.qkv.row_pos[row];
      sm.pos[cc] = pos;
      sm.page[cc] = g.qkv.page_table[(size_t)g.qkv.row_task[row] * g.qkv.pt_stride + (pos >> 4)];
    }
    if (g.rs_ss) {
      float t = 0.f;
      const float* rs = g.rs_ss + (size_t)n * g.rs_tiles;
      if (g.rs_tiles == 32 && ((uintptr_t)rs & 15) == 0) {  // d = 4096: all 8 loads in flight
        float4 r4[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) r4[i] = __ldcg(reinterpret_cast<const float4*>(rs) + i);
#pragma unroll
        for (int i = 0; i < 8; ++i) t = (((t + r4[i].x) + r4[i].y) + r4[i].z) + r4[i].w;
      } else {
        for (int i = 0; i < g.rs_tiles; ++i) t += __ldcg(rs + i);
      }
      sm.inv[cc] = rsqrtf(t / (float)g.K + 1e-5f);
    }
  }
  epi_bar(sm.bar);
  if (ce - cb > 16 || !allow_pre) return false;
  const int m = m_tile * 128 + et;
  // all (<= 16 columns) loads in flight at once, then the shared stores (a serial
  // load -> store loop paid one L2 round trip per column: the top stall of the O projection)
  if constexpr (MODE == EPI_RESID) {
    float v[16];
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      const int c = cb + k;
      v[k] = (c < ce && m < g.M && n0 + c < g.N) ? __ldcg(g.x + (size_t)(n0 + c) * g.M + m) : 0.f;
    }
#pragma unroll
    for (int k = 0; k < 16; ++k)
      if (cb + k < ce) sm.xp[k * 128 + et] = v[k];
    return true;
  } else if constexpr (MODE == EPI_QKV) {
    const int half = g.qkv.hd >> 1;
    if (et < 64) {  // cos / sin of the rotation (position of the column, frequency i)
      const int i = et % half;
      float vc[16], vs[16];
#pragma unroll
      for (int k = 0; k < 16; ++k) {
        const int c = cb + k;
        const bool ok = c < ce && n0 + c < g.N;
        const int pos = ok ? sm.pos[c] : 0;
        vc[k] = ok ? __ldg(g.qkv.cos + (size_t)pos * half + i) : 0.f;
        vs[k] = ok ? __ldg(g.qkv.sin + (size_t)pos * half + i) : 0.f;
      }
#pragma unroll
      for (int k = 0; k < 16; ++k)
        if (cb + k < ce) {
          sm.xp[k * 64 + et] = vc[k];
          sm.xp[1024 + k * 64 + et] = vs[k];
        }
    }
    return true;
  }
  return false;
}

__device__ __forceinline__ void cluster_arrive() { asm volatile("barrier.cluster.arrive.aligned;" ::: "memory"); }
__device__ __forceinline__ void cluster_wait() { asm volatile("barrier.cluster.wait.aligned;" ::: "memory"); }
// DSMEM push: bulk copy of `bytes` from this CTA's shared memory to the same-offset-space
// address `dst` of another CTA of the cluster, completing on that CTA's mbarrier `bar`
// (both cluster addresses from mapa)
__device__ __forceinline__ void bulk_s2cluster(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
      "r"(smem_u32(src)), "r"(bytes), "r"(bar)
      : "memory");
}

template <int BN, int MODE>
__global__ void __launch_bounds__(kGemmThreads, GemmCfg<BN>::CTAS_PER_SM)
    k_gemm_tc(const __grid_constant__ TmaMap tmB, GemmArgs g) {
  using C = GemmCfg<BN>;
  extern __shared__ unsigned char smem_raw[];
  unsigned char* smem = (unsigned char*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  unsigned char* sA = smem;
  unsigned char* sB = smem + C::STAGES * C::A_BYTES;
  unsigned char* ctl = smem + C::STAGES * C::STAGE;
  uint64_t* full = reinterpret_cast<uint64_t*>(ctl);
  uint64_t* empty = full + C::STAGES;
  uint64_t* done = empty + C::STAGES;
  uint64_t* recv_bar = done + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(recv_bar + 1);
  // after the mainloop the ring holds this CTA's fp32 partial tile P [BN][128] (column
  // major) and, with the push reduction, the receive slots [S][slot_cols][128]
  float* P = reinterpret_cast<float*>(smem);
  float* R = P + BN * 128;
  EpiSmem sm;
  sm.pos = reinterpret_cast<int*>(ctl + 512);
  sm.page = sm.pos + BN;
  sm.inv = reinterpret_cast<float*>(sm.page + BN);
  sm.redv = reinterpret_cast<float*>(ctl + 512 + C::META);
  sm.redi = reinterpret_cast<int*>(sm.redv + 4 * BN);
  sm.bn = BN;
  sm.xp = reinterpret_cast<float*>(ctl + 512 + C::META + C::RED);
  sm.xp_sin = 1024;
  __shared__ long long s_mark[9];  // clock64 phase marks (SM cycles), RT_FLAG_TRACE
  sm.mark = s_mark;

  TraceScope tr(TK_GEMM | ((uint32_t)MODE << 8) | (gridDim.x << 16));
  __shared__ unsigned long long s_tdone;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int S = gridDim.x;                 // cluster = the S split-K CTAs of one tile
  const int rank = S > 1 ? (int)cluster_rank() : 0;
  // several n-tiles (prefill rows > BN): the n-tiles of one m-tile are adjacent in the grid
  // (blockIdx.y) so they run together and the second reads the weight tile from L2
  const int lt = g.tile0 + (int)blockIdx.y;  // linear tile, n-tiles of one m-tile adjacent
  const int m_tile = lt / g.n_tiles, n_tile = lt - (lt / g.n_tiles) * g.n_tiles;
  const int kb0 = (int)(((long long)g.kb_total * rank) / S);
  const int kb1 = (int)(((long long)g.kb_total * (rank + 1)) / S);
  const int nkb = kb1 - kb0;
  const int n0 = n_tile * BN;
  const int cb = (BN * rank) / S, ce = (BN * (rank + 1)) / S;  // columns this CTA finishes
  const int slot_cols = (BN + S - 1) / S;
  const bool push = C::PUSH && S > 1;
  bool pre = false;  // epilogue inputs prefetched into sm.xp

  if (warp == 0 && lane == 0) {
    prefetch_tmap(&tmB);
    for (int s = 0; s < C::STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(done, 1);
    mbar_init(recv_bar, 1);
    fence_mbar_init();
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(C::TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  // EPI_QKV: dependents (the decode attention) may launch only once this kernel has passed
  // its own dependency wait — the attention reads the round's row metadata before its wait,
  // which is safe only if every kernel before it has completed (PDL)
  constexpr bool QKV_LIKE = MODE == EPI_QKV || MODE == EPI_PART;
  // EPI_PART: no split-K exchange at all — every split writes its raw partial
  constexpr bool PART = MODE == EPI_PART;
  if (!QKV_LIKE && threadIdx.x == 0) pdl_trigger();

  if (warp == 0) {
    if (lane == 0) {
      // weights do not depend on the previous kernel: request the first stages' W tiles
      // before waiting for it (programmatic dependent launch)
      const int pre_k = min(C::STAGES, nkb);
      // UMMA-tiled weights: k-block kb of m-tile mt is one contiguous 16 KiB SW128 image
      const bf16* wt = g.w + ((size_t)m_tile * g.kb_total + kb0) * (128 * kBK);
      const uint64_t pol = g.l2_evict_first ? l2_policy_evict_first() : 0ull;
      for (int i = 0; i < pre_k; ++i) {
        mbar_arrive_expect_tx(&full[i], C::STAGE);
        bulk_g2s_hint(sA + i * C::A_BYTES, wt + (size_t)i * (128 * kBK), C::A_BYTES, &full[i], pol);
      }
      pdl_wait();
      if (QKV_LIKE) pdl_trigger();
      tr.ready();
      for (int i = 0; i < pre_k; ++i)
        tma_load_2d(sB + i * C::B_BYTES, &tmB, (kb0 + i) * kBK, n0, &full[i]);
      for (int i = pre_k; i < nkb; ++i) {
        const int s = i % C::STAGES;
        const uint32_t ph = (uint32_t)((i / C::STAGES) & 1);
        mbar_wait(&empty[s], ph ^ 1u);
        mbar_arrive_expect_tx(&full[s], C::STAGE);
        bulk_g2s_hint(sA + s * C::A_BYTES, wt + (size_t)i * (128 * kBK), C::A_BYTES, &full[s], pol);
        tma_load_2d(sB + s * C::B_BYTES, &tmB, (kb0 + i) * kBK, n0, &full[s]);
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idesc = umma_idesc(128, BN);
      for (int i = 0; i < nkb; ++i) {
        const int s = i % C::STAGES;
        mbar_wait(&full[s], (uint32_t)((i / C::STAGES) & 1));
        tc_fence_after();
        const uint32_t a0 = smem_u32(sA + s * C::A_BYTES);
        const uint32_t b0 = smem_u32(sB + s * C::B_BYTES);
#pragma unroll
        for (int k = 0; k < kBK / 16; ++k)
          umma_f16(tmem, umma_desc_sw128(a0 + k * 32), umma_desc_sw128(b0 + k * 32), idesc,
                   (i > 0 || k > 0) ? 1u : 0u);
        umma_commit(&empty[s]);
      }
      umma_commit(done);
    }
    __syncwarp();
  } else {
    pdl_wait();
    const int q = warp & 3;
    const int et = q * 32 + lane;  // tile row owned by this thread
    const uint32_t tb = tmem + ((uint32_t)(q * 32) << 16);
    // per-column metadata + epilogue inputs of the columns this CTA finishes, while the
    // mainloop runs
    pre = column_meta<MODE>(g, sm, m_tile, n0, cb, ce, et);
    mbar_wait(done, 0);
    tc_fence_after();
    if (et == 0) {
      s_tdone = gtimer();
      const long long t = clock64();
#pragma unroll
      for (int i = 0; i < 9; ++i) s_mark[i] = t;
    }
    if constexpr (PART) {  // raw partial of split `rank` -> part[rank][n][m] (coalesced over m)
      const int m = m_tile * 128 + et;
      float* dst = g.part + ((size_t)rank * g.part_ld_n + n0) * g.M + m;
#pragma unroll 1
      for (int c0 = 0; c0 < BN && n0 + c0 < g.N; c0 += 16) {
        float v[16];
        tmem_ld16(tb + c0, v);
#pragma unroll
        for (int j = 0; j < 16; ++j)
          if (m < g.M && n0 + c0 + j < g.N) __stcg(dst + (size_t)(c0 + j) * g.M, v[j]);
      }
    }
    // split-K push: arrive on the cluster barrier as soon as this CTA's MMAs are done (its
    // ring may then receive the peers' slices) and park the accumulator while the slower
    // CTAs finish; the park writes P, the peers write the receive slots R (disjoint).  Pull
    // (the peers READ P over DSMEM after the barrier): arrive only once P is parked — an
    // early arrive there let a peer read a half-written P (intermittent wrong sums, found by
    // a run-to-run determinism check, tools/determinism_check.py)
    if (!PART && S > 1 && push) cluster_arrive();
#pragma unroll 1
    for (int c0 = 0; c0 < (PART ? 0 : BN); c0 += 16) {  // park the accumulator in shared memory
      float v[16];
      tmem_ld16(tb + c0, v);
#pragma unroll
      for (int j = 0; j < 16; ++j) P[(c0 + j) * 128 + et] = v[j];
    }
    if (push) fence_proxy_async();  // P is read by the bulk-copy (async) proxy
    if (!PART && S > 1 && !push) cluster_arrive();
    EPI_MARK(1);
    if (!PART && S > 1) cluster_wait();
  }
  // ---- cluster split-K: CTA `rank` finishes columns [cb, ce) of the tile.  The barrier
  // also certifies that every CTA's mainloop is over (its ring is free for the slices).
  if (!PART && S > 1 && warp < 2) {  // (the epilogue warps arrived / waited above)
    __syncwarp();
    cluster_arrive();
    cluster_wait();
  }
  if (!PART && warp >= 2) {
    const int et = (warp & 3) * 32 + lane;
    EPI_MARK(2);
    if (S > 1 && push) {
      // push: each CTA sends the column slice of every other rank straight into that
      // rank's receive slot [my rank] (one bulk copy per peer, TMA engine), then sums the
      // S slices of its own columns from local shared memory
      if (et == 0) {
        mbar_arrive_expect_tx(recv_bar, (uint32_t)((S - 1) * (ce - cb) * 512));
        const uint32_t rslot = smem_u32(R + (size_t)rank * slot_cols * 128);
        for (int r = 0; r < S; ++r) {
          if (r == rank) continue;
          const int rb = (BN * r) / S, re = (BN * (r + 1)) / S;
          bulk_s2cluster(dsmem_addr(rslot, (uint32_t)r), P + (size_t)rb * 128, (uint32_t)((re - rb) * 512),
                         dsmem_addr(smem_u32(recv_bar), (uint32_t)r));
        }
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      }
      mbar_wait(recv_bar, 0);
    }
    EPI_MARK(3);
    const TileSrc ts{P, R, smem_u32(P), S, rank, slot_cols, cb, S == 1 ? 0 : (push ? 1 : 2)};
    epilogue<MODE>(g, sm, ts, m_tile, n0, cb, ce, et, pre);
    if (push && et == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
    EPI_MARK(8);
  }
  if (!PART && S > 1 && !push) {  // keep shared memory alive until every CTA has read it
    __syncwarp();
    cluster_arrive();
    cluster_wait();
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x == 0) {
    tr.aux(s_tdone);
    // SM-cycle durations of the 8 phases after the accumulator is complete (clock64; the
    // %globaltimer granularity is too coarse for them), two per 64-bit field: park |
    // cluster barrier | slices received | - | - | epilogue loop | final reduction | exit
    auto dd = [&](int i) {
      const long long d = s_mark[i + 1] - s_mark[i];
      return (unsigned long long)(uint32_t)(d > 0 ? d : 0);
    };
    trace_phase(TK_PHASE | TK_GEMM | ((uint32_t)MODE << 8) | (gridDim.x << 16), dd(0) | (dd(1) << 32),
                dd(2) | (dd(3) << 32), dd(4) | (dd(5) << 32), dd(6) | (dd(7) << 32));
  }
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(C::TMEM_COLS));
  }
}

// ============================================================ hybrid DP + stream-K projection
// Rounds with prompt rows run the projections at N = 130 .. 8192 rows, where the GEMM is
// tensor-bound and one tile per CTA quantises badly on 148 SMs (gate/up at N = 256: 224
// tiles = 1.5 waves; N = 352 on 192-wide tiles: 448 tiles = 3.03 waves) and pays a pipeline
// fill + an unoverlapped epilogue per tile.  k_gemm_sk: one persistent CTA per SM.  Tiles
// (n-tiles of an m-tile adjacent) are split into data-parallel whole tiles, round-robin over
// the CTAs (all full waves but one), and a stream-K part (the last full wave + the partial
// one, so every stream-K tile has <= 3 contributors) whose k-block iterations are split
// evenly over the CTAs.  Each segment accumulates in one of two TMEM buffers, so a
// segment's epilogue overlaps the next segment's MMAs; the ring stays full across
// segments.  A stream-K segment that is not a whole tile stores its fp32 partial to the
// CTA's workspace slot (0: its first stream-K tile, 1: its last) and takes a ticket; the
// last contributor sums the partials in contributor order (deterministic) and runs the
// fused epilogue in column chunks staged through shared memory.
namespace sk {
// stream-K k-block iterations: I = tiles * kb; CTA c owns [q0(c), q0(c + 1))
__host__ __device__ inline int q0(long long I, int c, int P) { return (int)((I * c) / P); }
// the CTA whose range contains iteration q (valid when I >= P: no empty ranges)
__host__ __device__ inline int owner(long long q, long long I, int P) { return (int)(((q + 1) * P - 1) / I); }
constexpr int A_BYTES = 128 * kBK * 2;
template <int BN>
struct Cfg {
  // ring depth: as many stages as fit beside the epilogue staging (the mainloop of these
  // tensor-bound prefill tiles is latency bound on the L2 / HBM round trip of each stage)
  static constexpr int STAGES = BN <= 160 ? 5 : 4;
  static constexpr int CHUNK = BN == 256 ? 32 : 64;      // epilogue columns per staging pass
  static constexpr int STG_BYTES = CHUNK * 128 * 4;
  static constexpr int B_BYTES = BN * kBK * 2;
  static constexpr int TMEM_COLS = 2 * BN <= 256 ? 256 : 512;
  static constexpr int CTL = 256;
  static constexpr int META = 3 * BN * 4;
  static constexpr int RED = 2 * 4 * BN * 4;
  static constexpr int SMEM = 1024 + STAGES * (A_BYTES + B_BYTES) + STG_BYTES + CTL + META + RED;
  static_assert(SMEM <= 227 * 1024, "hybrid stream-K smem");
};
// the segment sequence of one CTA: its PARTIAL stream-K segments first (last one first: it
// is the head of a tile whose tail the next CTA computes at its start, so both partials of a
// tile are ready early and the fixup overlaps the whole tiles that follow), then its
// data-parallel tiles, then its whole stream-K tiles
struct Sched {
  static constexpr int MAXS = 8;
  int P, cta, kbt, n_tiles;
  int dp_tiles, dp_mine;     // data-parallel tiles (a multiple of P) and this CTA's count
  long long I_sk;            // stream-K iterations (sk tiles x kbt)
  int qa, qb;                // this CTA's stream-K range
  int ns, sl[MAXS], sh[MAXS], st[MAXS];  // stream-K segments in range order (lo, hi, sk tile)
  int np, order[MAXS];       // partial segments first (reversed), then whole ones
  __device__ void init(int P_, int cta_, int kbt_, int T, int n_tiles_, bool all_sk) {
    P = P_;
    cta = cta_;
    kbt = kbt_;
    n_tiles = n_tiles_;
    const int sk_tiles = (all_sk || T <= P) ? T : (T % P) + P;
    dp_tiles = T - sk_tiles;
    dp_mine = dp_tiles / P;
    I_sk = (long long)sk_tiles * kbt;
    qa = q0(I_sk, cta, P);
    qb = q0(I_sk, cta + 1, P);
    ns = 0;
    for (int q = qa; q < qb && ns < MAXS;) {
      const int t = q / kbt;
      sl[ns] = q - t * kbt;
      sh[ns] = min(qb - t * kbt, kbt);
      st[ns] = t;
      q = t * kbt + sh[ns];
      ++ns;
    }
    np = 0;
    for (int i = ns - 1; i >= 0; --i)
      if (sl[i] != 0 || sh[i] != kbt) order[np++] = i;
    int k = np;
    for (int i = 0; i < ns; ++i)
      if (sl[i] == 0 && sh[i] == kbt) order[k++] = i;
  }
  struct Seg {
    int tile, lo, hi;   // global tile index, k-block range
    int sk_t;           // stream-K tile index (-1: data-parallel)
  };
  // step i: [0, np) partial stream-K, [np, np + dp_mine) data-parallel, then whole stream-K
  __device__ bool first(Seg& g, int& i, int& unused) const {
    i = 0;
    unused = 0;
    return next(g, i, unused);
  }
  __device__ bool next(Seg& g, int& i, int&) const {
    if (i >= ns + dp_mine) return false;
    if (i >= np && i < np + dp_mine) {
      g.tile = cta + (i - np) * P;
      g.lo = 0;
      g.hi = kbt;
      g.sk_t = -1;
    } else {
      const int j = order[i < np ? i : i - dp_mine];
      g.sk_t = st[j];
      g.tile = dp_tiles + st[j];
      g.lo = sl[j];
      g.hi = sh[j];
    }
    ++i;
    return true;
  }
};
}  // namespace sk

struct SkArgs {
  int P;             // CTAs
  int n_tiles;       // tiles along N (BN rows each)
  float* ws;         // [P][2][BN][128] partial tiles
  unsigned* cnt;     // [m_tiles * n_tiles] zero-initialised, self-resetting tickets
  int all_sk;        // every tile stream-K (no data-parallel part)
  // CTA-pair kernel, data-parallel order: pair-tiles [head, PT) (the partial last round) run
  // as sub_s sub-tiles of kPairSubW columns each, one per pair (0: no sub-tiles)
  int head, sub_s;
};

template <int BN, int MODE>
__global__ void __launch_bounds__(kGemmThreads, 1)
    k_gemm_sk(const __grid_constant__ TmaMap tmB, GemmArgs g, SkArgs a) {
  using C = sk::Cfg<BN>;
  using namespace sk;
  constexpr int CHUNK = C::CHUNK;
  constexpr int STAGES = C::STAGES;
  extern __shared__ unsigned char smem_raw[];
  unsigned char* smem = (unsigned char*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  unsigned char* sA = smem;
  unsigned char* sB = smem + STAGES * A_BYTES;
  float* stg = reinterpret_cast<float*>(sB + STAGES * C::B_BYTES);
  unsigned char* ctl = reinterpret_cast<unsigned char*>(stg) + C::STG_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(ctl);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 2;
  uint64_t* fxbar = tempty + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(fxbar + 1);
  int* s_last = reinterpret_cast<int*>(tmem_slot + 1);
  EpiSmem sm;
  sm.pos = reinterpret_cast<int*>(ctl + C::CTL);
  sm.page = sm.pos + BN;
  sm.inv = reinterpret_cast<float*>(sm.page + BN);
  sm.redv = reinterpret_cast<float*>(ctl + C::CTL + C::META);
  sm.redi = reinterpret_cast<int*>(sm.redv + 4 * BN);
  sm.bn = BN;
  sm.xp = stg;  // unused (pre = false)
  sm.xp_sin = 0;
  __shared__ long long s_mark[9];
  sm.mark = s_mark;

  TraceScope tr(TK_GEMM | ((uint32_t)MODE << 8) | (1u << 16));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int cta = blockIdx.x;
  const int kbt = g.kb_total;
  Sched S;
  S.init(a.P, cta, kbt, g.m_tiles * a.n_tiles, a.n_tiles, a.all_sk != 0);

  if (warp == 0 && lane == 0) {
    prefetch_tmap(&tmB);
    for (int i = 0; i < STAGES; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tfull[i], 1);
      mbar_init(&tempty[i], 1);
    }
    mbar_init(fxbar, 1);
    fence_mbar_init();
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(C::TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  if (MODE != EPI_QKV && threadIdx.x == 0) pdl_trigger();  // EPI_QKV: after the wait (k_gemm_tc)

  if (warp == 0) {
    if (lane == 0) {
      bool waited = false;
      int n = 0, d, q;
      Sched::Seg sg;
      for (bool ok = S.first(sg, d, q); ok; ok = S.next(sg, d, q)) {
        const int m_tile = sg.tile / a.n_tiles, n_tile = sg.tile - m_tile * a.n_tiles;
        for (int kb = sg.lo; kb < sg.hi; ++kb, ++n) {
          const int st = n % STAGES;
          if (n >= STAGES) mbar_wait(&empty[st], (uint32_t)(((n / STAGES) & 1) ^ 1));
          mbar_arrive_expect_tx(&full[st], A_BYTES + C::B_BYTES);
          bulk_g2s(sA + st * A_BYTES, g.w + ((size_t)m_tile * kbt + kb) * (128 * kBK), A_BYTES, &full[st]);
          if (!waited) {  // weights before the previous kernel finishes, activations after
            pdl_wait();
            if (MODE == EPI_QKV) pdl_trigger();
            tr.ready();
            waited = true;
          }
          tma_load_2d(sB + st * C::B_BYTES, &tmB, kb * kBK, n_tile * BN, &full[st]);
        }
      }
      if (!waited) {
        pdl_wait();
        if (MODE == EPI_QKV) pdl_trigger();
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idesc = umma_idesc(128, BN);
      int n = 0, seg = 0, d, q;
      Sched::Seg sg;
      for (bool ok = S.first(sg, d, q); ok; ok = S.next(sg, d, q)) {
        const int buf = seg & 1;
        if (seg >= 2) mbar_wait(&tempty[buf], (uint32_t)(((seg >> 1) - 1) & 1));
        tc_fence_after();
        const uint32_t acc = tmem + (uint32_t)(buf * BN);
        for (int kb = sg.lo; kb < sg.hi; ++kb, ++n) {
          const int st = n % STAGES;
          mbar_wait(&full[st], (uint32_t)((n / STAGES) & 1));
          tc_fence_after();
          const uint32_t a0 = smem_u32(sA + st * A_BYTES);
          const uint32_t b0 = smem_u32(sB + st * C::B_BYTES);
#pragma unroll
          for (int k = 0; k < kBK / 16; ++k)
            umma_f16(acc, umma_desc_sw128(a0 + k * 32), umma_desc_sw128(b0 + k * 32), idesc,
                     (kb > sg.lo || k > 0) ? 1u : 0u);
          umma_commit(&empty[st]);
        }
        umma_commit(&tfull[buf]);
        ++seg;
      }
    }
    __syncwarp();
  } else {
    pdl_wait();
    const int et = (warp & 3) * 32 + lane;
    const uint32_t tb = tmem + ((uint32_t)((warp & 3) * 32) << 16);
    const int first_sk = S.qa / kbt;
    uint32_t fx_phase = 0u;
    int seg = 0, d, q;
    Sched::Seg sg;
    for (bool ok = S.first(sg, d, q); ok; ok = S.next(sg, d, q)) {
      const int buf = seg & 1;
      const int m_tile = sg.tile / a.n_tiles, n_tile = sg.tile - m_tile * a.n_tiles;
      const int n0 = n_tile * BN;
      int nc = 1, c_first = 0;
      if (sg.sk_t >= 0) {
        c_first = owner((long long)sg.sk_t * kbt, S.I_sk, S.P);
        nc = owner((long long)(sg.sk_t + 1) * kbt - 1, S.I_sk, S.P) - c_first + 1;
      }
      mbar_wait(&tfull[buf], (uint32_t)((seg >> 1) & 1));
      tc_fence_after();
      epi_bar();  // the previous segment's epilogue is done with the staging buffer / sm
      bool run = true;
      const uint32_t tacc = tb + (uint32_t)(buf * BN);
      if (nc > 1) {
        float* mine = a.ws + ((size_t)cta * 2 + (sg.sk_t == first_sk ? 0 : 1)) * (BN * 128);
#pragma unroll 1
        for (int c0 = 0; c0 < BN; c0 += 16) {
          float v[16];
          tmem_ld16(tacc + (uint32_t)c0, v);
#pragma unroll
          for (int i = 0; i < 16; ++i) __stcg(mine + (size_t)(c0 + i) * 128 + et, v[i]);
        }
        tc_fence_before();
        __threadfence();
        epi_bar();
        if (et == 0) {
          mbar_arrive(&tempty[buf]);
          const unsigned old = atomicAdd(a.cnt + sg.tile, 1u);
          *s_last = (old == (unsigned)(nc - 1)) ? 1 : 0;
        }
        epi_bar();
        run = *s_last != 0;
        if (run) {
          __threadfence();
          if (et == 0) {
            a.cnt[sg.tile] = 0u;
            asm volatile("fence.proxy.async.global;" ::: "memory");
          }
        }
      }
      if (run) {
        column_meta<MODE>(g, sm, m_tile, n0, 0, BN, et);  // per-column metadata of this tile's rows
        const TileSrc ts0{nullptr, nullptr, 0u, 1, 0, BN, 0, 0};
#pragma unroll 1
        for (int cb = 0; cb < BN; cb += CHUNK) {
          const int ce = min(BN, cb + CHUNK);
          if (nc == 1) {  // whole tile: TMEM -> staging
#pragma unroll 1
            for (int c0 = cb; c0 < ce; c0 += 16) {
              float v[16];
              tmem_ld16(tacc + (uint32_t)c0, v);
#pragma unroll
              for (int i = 0; i < 16; ++i) stg[(c0 - cb + i) * 128 + et] = v[i];
            }
          } else {  // sum the nc partials of columns [cb, ce) in contributor order
            float acc[CHUNK];
#pragma unroll
            for (int c = 0; c < CHUNK; ++c) acc[c] = 0.f;
            const uint32_t bytes = (uint32_t)((ce - cb) * 512);
            for (int r = 0; r < nc; ++r) {
              const int c = c_first + r;
              if (et == 0) {
                const int fs = q0(S.I_sk, c, S.P) / kbt;
                const float* src = a.ws + ((size_t)c * 2 + (sg.sk_t == fs ? 0 : 1)) * (BN * 128) + (size_t)cb * 128;
                mbar_arrive_expect_tx(fxbar, bytes);
                bulk_g2s(stg, src, bytes, fxbar);
              }
              mbar_wait(fxbar, fx_phase);
              fx_phase ^= 1u;
#pragma unroll
              for (int cc = 0; cc < CHUNK; ++cc)
                if (cb + cc < ce) acc[cc] += stg[cc * 128 + et];
              epi_bar();  // the staging buffer is free for the next partial
            }
#pragma unroll
            for (int cc = 0; cc < CHUNK; ++cc)
              if (cb + cc < ce) stg[cc * 128 + et] = acc[cc];
          }
          epi_bar();
          TileSrc ts = ts0;
          ts.P = stg - (size_t)cb * 128;  // the epilogue indexes absolute columns
          epilogue<MODE>(g, sm, ts, m_tile, n0, cb, ce, et, false);
          epi_bar();
        }
        if (nc == 1) {
          tc_fence_before();
          if (et == 0) mbar_arrive(&tempty[buf]);
        }
      }
      ++seg;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(C::TMEM_COLS));
  }
}

// ------------------------------------------------------- CTA-pair (cta_group::2) path
// Prefill projections (N > 128 activation rows) are tensor-bound, and with one SM per
// 128 x BN tile they are bound by SHARED-MEMORY bandwidth: every k-block writes A (16 KB)
// and B (BN x 128 B) into shared memory by TMA and the MMA reads both back, ~200 B per
// clock at BN = 192 against ~128 B per clock per SM (ncu: 49 % tensor-pipe active, nothing
// else saturated, profiles/r01_ncu_gemm_prefill384_full.json).  A CTA pair on the two SMs
// of a TPC issues ONE tcgen05.mma.cta_group::2 with M = 256: each CTA holds the 128 weight
// rows of its own m-tile (A) but only HALF of the BN activation rows (B), the tensor core
// reading the other half from the peer — per SM the B traffic halves (BN = 256: 32 KB per
// k-block instead of 48 KB).  Persistent, data-parallel: pair p takes the pair-tiles
// p, p + n_pairs, ...; TMEM holds two BN-column accumulators per CTA (the epilogue of tile
// i overlaps the mainloop of tile i + 1).
//   both CTAs, warp 0 lane 0: TMA loads of its A tile (the pre-tiled weight image through a
//     2-D map, no swizzle: the bytes are already SW128) and its half of X, both completing
//     on the LEADER's full barrier (cp.async.bulk.tensor .cta_group::2); the leader alone
//     expects the transaction bytes of both CTAs;
//   leader, warp 1 lane 0: tcgen05.mma.cta_group::2 (M = 256, N = BN, K = 16), commits
//     multicast to both CTAs' empty / accumulator-full barriers;
//   both CTAs, warps 2..5: epilogue of their own 128 output features (the same fused
//     epilogue as the single-SM kernels), then release the accumulator buffer on the
//     leader's barrier (count 2: one arrival per CTA).
namespace sm2 {
template <int BN>
struct Cfg {
  static constexpr int HB = BN / 2;  // activation rows per CTA
  static constexpr int A_BYTES = 128 * kBK * 2;
  static constexpr int B_BYTES = HB * kBK * 2;
  static constexpr int STAGE = A_BYTES + B_BYTES;
#ifndef RT_PAIR_CHUNK
#define RT_PAIR_CHUNK 16
#endif
  static constexpr int CHUNK = RT_PAIR_CHUNK;          // epilogue columns per staging pass (per group)
  static constexpr int STG_BYTES = 2 * CHUNK * 128 * 4;  // one staging buffer per epilogue group
  static constexpr int TMEM_COLS = 2 * BN <= 256 ? 256 : 512;
  static constexpr int CTL = 256;
  static constexpr int META = 3 * BN * 4;
  static constexpr int RED = 2 * 4 * BN * 4;
  static constexpr int FIXED = 1024 + STG_BYTES + CTL + META + RED;
  static constexpr int FIT = (227 * 1024 - FIXED) / STAGE;
  static constexpr int STAGES = FIT > 8 ? 8 : FIT;
  static constexpr int SMEM = FIXED + STAGES * STAGE;
  static_assert(STAGES >= 4, "CTA-pair ring depth");
};
}  // namespace sm2

__device__ __forceinline__ void tma_load_2d_pair(void* dst, const void* tmap, int c0, int c1, uint32_t bar_cluster) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, "
      "%3}], [%4];" ::"r"(smem_u32(dst)),
      "l"(tmap), "r"(c0), "r"(c1), "r"(bar_cluster)
      : "memory");
}
__device__ __forceinline__ void umma_f16_pair(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                              uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}
// arrive on the barrier at this offset in every CTA of `mask` once the issued MMAs complete
__device__ __forceinline__ void umma_commit_pair(uint64_t* bar, uint16_t mask) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          smem_u32(bar)),
      "h"(mask)
      : "memory");
}
__device__ __forceinline__ void mbar_arrive_cluster(uint32_t bar_cluster) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(bar_cluster) : "memory");
}

// work of one pair: data-parallel pair-tiles (pair, pair + n_pairs, ...); the partial last
// round may run as sub-tiles of kPairSubW columns, one per pair
constexpr int kPairSubW = 64;  // sub-tile width of the partial last round (32 rows per CTA)
struct PSeg {
  int tile;  // pair-tile
  int sub;   // sub-tile (columns [sub * kPairSubW, +kPairSubW) of the pair-tile), -1: whole
};
struct PairSeq {
  int pair, n_pairs, PT, head, sub_s;
  __device__ void init(int pair_, int n_pairs_, int PT_, int head_, int sub_s_) {
    pair = pair_;
    n_pairs = n_pairs_;
    PT = PT_;
    head = sub_s_ > 0 ? head_ : PT_;
    sub_s = sub_s_;
  }
  __device__ bool next(PSeg& g, int& i) const {
    g.sub = -1;
    const int t = pair + i * n_pairs;
    if (t < head) {
      g.tile = t;
      ++i;
      return true;
    }
    // the partial last round: sub-tile u = pair of the tail pair-tiles' sub_s sub-tiles
    if (sub_s == 0 || t - pair != head || pair >= (PT - head) * sub_s) return false;
    g.tile = head + pair / sub_s;
    g.sub = pair % sub_s;
    ++i;
    return true;
  }
};

template <int BN, int MODE>
__global__ void __launch_bounds__(kDecThreads, 1)
    k_gemm_2sm(const __grid_constant__ TmaMap tmA, const __grid_constant__ TmaMap tmB,
               const __grid_constant__ TmaMap tmBs, GemmArgs g, SkArgs a) {
  using C = sm2::Cfg<BN>;
  constexpr int STAGES = C::STAGES, CHUNK = C::CHUNK;
  extern __shared__ unsigned char smem_raw[];
  unsigned char* smem = (unsigned char*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  unsigned char* sA = smem;
  unsigned char* sB = smem + STAGES * C::A_BYTES;
  float* stg = reinterpret_cast<float*>(sB + STAGES * C::B_BYTES);
  unsigned char* ctl = reinterpret_cast<unsigned char*>(stg) + C::STG_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(ctl);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  EpiSmem sm;
  sm.pos = reinterpret_cast<int*>(ctl + C::CTL);
  sm.page = sm.pos + BN;
  sm.inv = reinterpret_cast<float*>(sm.page + BN);
  sm.redv = reinterpret_cast<float*>(ctl + C::CTL + C::META);
  sm.redi = reinterpret_cast<int*>(sm.redv + 4 * BN);
  sm.bn = BN;
  sm.xp = stg;  // unused (pre = false)
  sm.xp_sin = 0;
  __shared__ long long s_mark[9];
  sm.mark = s_mark;

  TraceScope tr(TK_GEMM | ((uint32_t)MODE << 8) | (2u << 16));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_rank();
  const int pair = blockIdx.x >> 1;
  const int kbt = g.kb_total;
  const int nt_n = a.n_tiles;
  const int PT = (g.m_tiles >> 1) * nt_n;
  PairSeq Q;
  Q.init(pair, a.P, PT, a.head, a.sub_s);

  if (warp == 0 && lane == 0) {
    prefetch_tmap(&tmA);
    prefetch_tmap(&tmB);
    prefetch_tmap(&tmBs);
    for (int i = 0; i < STAGES; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tfull[i], 1);
      mbar_init(&tempty[i], 4);  // one arrival per epilogue group of each CTA
    }
    fence_mbar_init();
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(C::TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  cluster_arrive();  // the peer's barriers are initialised before anyone signals them
  cluster_wait();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  if (MODE != EPI_QKV && threadIdx.x == 0) pdl_trigger();  // EPI_QKV: after the wait (k_gemm_tc)

  if (warp == 0) {
    if (lane == 0) {
      const uint32_t full0 = dsmem_addr(smem_u32(full), 0);  // the leader's full barriers
      bool waited = false;
      int n = 0, i = 0;
      PSeg sg;
      while (Q.next(sg, i)) {
        const int mp = sg.tile / nt_n, nt = sg.tile - mp * nt_n;
        const int m_tile = 2 * mp + (int)rank;
        const bool sub = sg.sub >= 0;
        // activation rows of this CTA: its half of the tile, or of the sub-tile
        const int brow = sub ? nt * BN + sg.sub * kPairSubW + (int)rank * (kPairSubW / 2) : nt * BN + (int)rank * C::HB;
        const uint32_t bytes = sub ? 2u * (C::A_BYTES + (kPairSubW / 2) * kBK * 2) : 2u * C::STAGE;
        for (int kb = 0; kb < kbt; ++kb, ++n) {
          const int st = n % STAGES;
          if (n >= STAGES) mbar_wait(&empty[st], (uint32_t)(((n / STAGES) & 1) ^ 1));
          if (rank == 0) mbar_arrive_expect_tx(&full[st], bytes);
          tma_load_2d_pair(sA + st * C::A_BYTES, &tmA, 0, (m_tile * kbt + kb) * 128, full0 + st * 8);
          if (!waited) {  // weights before the previous kernel finishes, activations after
            pdl_wait();
            if (MODE == EPI_QKV) pdl_trigger();
            tr.ready();
            waited = true;
          }
          tma_load_2d_pair(sB + st * C::B_BYTES, sub ? &tmBs : &tmB, kb * kBK, brow, full0 + st * 8);
        }
      }
      if (!waited) {
        pdl_wait();
        if (MODE == EPI_QKV) pdl_trigger();
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    if (rank == 0 && lane == 0) {
      int n = 0, seg = 0, i = 0;
      PSeg sg;
      for (; Q.next(sg, i); ++seg) {
        const uint32_t idesc = sg.sub >= 0 ? umma_idesc(256, kPairSubW) : umma_idesc(256, BN);
        const int buf = seg & 1;
        if (seg >= 2) mbar_wait(&tempty[buf], (uint32_t)(((seg >> 1) - 1) & 1));
        tc_fence_after();
        const uint32_t acc = tmem + (uint32_t)(buf * BN);
        for (int kb = 0; kb < kbt; ++kb, ++n) {
          const int st = n % STAGES;
          mbar_wait(&full[st], (uint32_t)((n / STAGES) & 1));
          tc_fence_after();
          const uint32_t a0 = smem_u32(sA + st * C::A_BYTES);
          const uint32_t b0 = smem_u32(sB + st * C::B_BYTES);
#pragma unroll
          for (int k = 0; k < kBK / 16; ++k)
            umma_f16_pair(acc, umma_desc_sw128(a0 + k * 32), umma_desc_sw128(b0 + k * 32), idesc,
                          (kb > 0 || k > 0) ? 1u : 0u);
          umma_commit_pair(&empty[st], 0x3);
        }
        umma_commit_pair(&tfull[buf], 0x3);
      }
    }
    __syncwarp();
  } else {
    // two epilogue groups of 4 warps (2-5, 6-9), both over the 128 TMEM lanes, taking
    // alternate CHUNK-column chunks of each tile with their own staging buffer: the last
    // tile's epilogue (not overlapped by a next mainloop) runs on 8 warps
    pdl_wait();
    const int grp = (warp - 2) >> 2;
    const int et = (warp & 3) * 32 + lane;
    const uint32_t tb = tmem + ((uint32_t)((warp & 3) * 32) << 16);
    const uint32_t tempty0 = dsmem_addr(smem_u32(tempty), 0);
    float* gstg = stg + (size_t)grp * CHUNK * 128;
    EpiSmem gsm = sm;
    gsm.bar = 1 + grp;
    gsm.mark = nullptr;
    long long c_wait = 0, c_park = 0, c_epi = 0;  // epilogue-warp cycle totals (trace phases)
    int seg = 0, i = 0;
    PSeg sg;
    for (; Q.next(sg, i); ++seg) {
      const long long c0w = clock64();
      const int buf = seg & 1;
      const int mp = sg.tile / nt_n, nt = sg.tile - mp * nt_n;
      const int m_tile = 2 * mp + (int)rank;
      const int n0 = nt * BN + (sg.sub >= 0 ? sg.sub * kPairSubW : 0);
      const int W = sg.sub >= 0 ? kPairSubW : BN;  // accumulator columns of this segment
      mbar_wait(&tfull[buf], (uint32_t)((seg >> 1) & 1));
      tc_fence_after();
      // both groups are done with the previous tile (staging, per-column metadata)
      asm volatile("bar.sync 3, 256;" ::: "memory");
      const long long c1w = clock64();
      c_wait += c1w - c0w;
      const uint32_t tacc = tb + (uint32_t)(buf * BN);
      if (grp == 0) column_meta<MODE>(g, sm, m_tile, n0, 0, W, et);  // (group barrier inside)
      asm volatile("bar.sync 3, 256;" ::: "memory");                // ... seen by group 1 too
      const TileSrc ts0{nullptr, nullptr, 0u, 1, 0, BN, 0, 0};
      const int n_ch = (W + CHUNK - 1) / CHUNK;
      const int my_last = ((n_ch - 1 - grp) >= 0) ? grp + 2 * ((n_ch - 1 - grp) / 2) : -1;  // last chunk of this group
#pragma unroll 1
      for (int ch = grp; ch < n_ch; ch += 2) {
        const int cb = ch * CHUNK;
        const int ce = min(W, cb + CHUNK);
        const long long cp0 = clock64();
        if constexpr (MODE == EPI_ARGMAX) {
          // lm_head: the column maxima are taken by a column scan of the staged tile, not by
          // cross-lane shuffle chains (one warp per SM sub-partition could not hide their
          // latency: 175 of the 282 us of the C3 lm_head were this epilogue).  Staging layout:
          // column c, rows 4q .. 4q + 3 at 16-byte chunk q ^ (c & 31) -> conflict-free for
          // both the row-per-thread writes and the column-per-thread 16-byte reads.
          const int m = m_tile * 128 + et;
#pragma unroll 1
          for (int c0 = cb; c0 < ce; c0 += 16) {
            float v[16];
            tmem_ld16(tacc + (uint32_t)c0, v);
#pragma unroll
            for (int k = 0; k < 16; ++k) {
              const int c = c0 - cb + k;
              gstg[c * 128 + ((((et >> 2) ^ (c & 31)) << 2) | (et & 3))] = v[k];
            }
            if (g.out && m < g.M)  // logits (parity mode only)
#pragma unroll
              for (int k = 0; k < 16; ++k)
                if (n0 + c0 + k < g.N) g.out[(size_t)(n0 + c0 + k) * g.M + m] = v[k];
          }
        } else {
#pragma unroll 1
          for (int c0 = cb; c0 < ce; c0 += 16) {  // TMEM -> staging
            float v[16];
            tmem_ld16(tacc + (uint32_t)c0, v);
#pragma unroll
            for (int k = 0; k < 16; ++k) gstg[(c0 - cb + k) * 128 + et] = v[k];
          }
        }
        c_park += clock64() - cp0;
        if (ch == my_last) {  // this group is done reading the accumulator: release its part
          tc_fence_before();
          epi_bar(gsm.bar);
          if (et == 0) {
            if (rank == 0) mbar_arrive(&tempty[buf]);
            else mbar_arrive_cluster(tempty0 + (uint32_t)buf * 8u);
          }
        }
        epi_bar(gsm.bar);
        const long long ce0 = clock64();
        if constexpr (MODE == EPI_ARGMAX) {
          // thread et scans quarter `hf` of the rows of column c (32 rows as 8 chunks of 4),
          // ascending -> the first maximum = the lowest vocabulary index (greedy, AMB: ties)
          constexpr int NHF = 128 / CHUNK < 4 ? 128 / CHUNK : 4;  // row parts (redv / redi hold 4)
          const int wc = ce - cb, c = et % CHUNK, hf = et / CHUNK;
          if (c < wc && hf < NHF) {
            float bv = -INFINITY;
            int br = 0;
            const float* col = gstg + (size_t)c * 128;
            const int rmax = g.M - m_tile * 128;  // rows beyond M (last m-tile) never win
            constexpr int QP = 32 / NHF;          // 16-byte chunks per part
#pragma unroll 4
            for (int q = QP * hf; q < QP * hf + QP; ++q) {
              const float4 x = *reinterpret_cast<const float4*>(col + ((q ^ (c & 31)) << 2));
              if (x.x > bv && 4 * q < rmax) { bv = x.x; br = 4 * q; }
              if (x.y > bv && 4 * q + 1 < rmax) { bv = x.y; br = 4 * q + 1; }
              if (x.z > bv && 4 * q + 2 < rmax) { bv = x.z; br = 4 * q + 2; }
              if (x.w > bv && 4 * q + 3 < rmax) { bv = x.w; br = 4 * q + 3; }
            }
            sm.redv[hf * BN + cb + c] = bv;
            sm.redi[hf * BN + cb + c] = m_tile * 128 + br;
          }
          epi_bar(gsm.bar);
          if (et < wc && n0 + cb + et < g.N) {
            float bv = sm.redv[cb + et];
            int bi = sm.redi[cb + et];
#pragma unroll
            for (int p = 1; p < NHF; ++p) {  // lower row parts win ties (lower index)
              const float ov = sm.redv[p * BN + cb + et];
              const int oi = sm.redi[p * BN + cb + et];
              if (ov > bv) {
                bv = ov;
                bi = oi;
              }
            }
            g.part_val[(size_t)m_tile * g.N + n0 + cb + et] = bv;
            g.part_idx[(size_t)m_tile * g.N + n0 + cb + et] = bi;
          }
        } else {
          TileSrc ts = ts0;
          ts.P = gstg - (size_t)cb * 128;  // the epilogue indexes absolute columns
          epilogue<MODE>(g, gsm, ts, m_tile, n0, cb, ce, et, false);
        }
        epi_bar(gsm.bar);
        c_epi += clock64() - ce0;
      }
      if (my_last < 0) {  // (a group without chunks in this tile still releases its part)
        tc_fence_before();
        if (et == 0) {
          if (rank == 0) mbar_arrive(&tempty[buf]);
          else mbar_arrive_cluster(tempty0 + (uint32_t)buf * 8u);
        }
      }
    }
    if (et == 0 && grp == 0) {  // trace: totals over this CTA's tiles (wait for the accumulator | park | epilogue)
      s_mark[0] = 0;
      s_mark[1] = c_wait;
      s_mark[2] = c_wait + c_park;
      s_mark[3] = c_wait + c_park + c_epi;
      for (int q = 4; q < 9; ++q) s_mark[q] = s_mark[3];
    }
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x == 0) {
    auto dd = [&](int i) {
      const long long d = s_mark[i + 1] - s_mark[i];
      return (unsigned long long)(uint32_t)(d > 0 ? d : 0);
    };
    trace_phase(TK_PHASE | TK_GEMM | ((uint32_t)MODE << 8) | (2u << 16), dd(0) | (dd(1) << 32),
                dd(2) | (dd(3) << 32), dd(4) | (dd(5) << 32), dd(6) | (dd(7) << 32));
  }
  cluster_arrive();  // no CTA leaves while its peer may still signal its barriers
  cluster_wait();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(C::TMEM_COLS));
  }
}

// ============================================================ decode CTA pairs, split-K
// Decode rounds of N <= 256 rows on the few-tile projections (QKV, O, down: 16-24 pair-tiles
// of 256 weight rows).  One SM per 128 x 256 tile is bound by SHARED-MEMORY bandwidth, not by
// HBM: per k-block TMA writes A (16 KB) + B (32 KB) and the MMA reads them back, ~192 B/clk
// against ~128 B/clk per SM (measured: QKV at N = 256 ran its mainloop at 3.6 TB/s).  Here a
// CTA pair (a cluster of 2) issues tcgen05.mma.cta_group::2 with M = 256: each CTA holds its
// 128 weight rows and HALF of the activation rows, so the B operand per SM halves (32 KB per
// k-block per SM: balanced with the MMA).  The K dimension is split over S pairs so that
// S x pair-tiles fill the SMs (QKV 24 x 3, O / down 16 x 4), one CTA per SM.
// Split-K reduction through L2, not DSMEM: clusters of 2S CTAs (6-8) did not all fit at once
// (two waves: down 73.6 us at C3 against 48 us before), so the S pairs of a tile are separate
// 2-CTA clusters.  Each CTA writes the column slices it does not own (fp32, st.global.cg) to
// the owner's slots of a workspace and publishes a per-(tile, half, pair) epoch flag (release);
// the owner (the CTA of pair q with the same half) spins on its S - 1 contributors' flags
// (acquire) and sums the S partials in pair order (deterministic).  Deadlock-free: S x PT <=
// 74 pairs, so every CTA is resident once the previous kernel has drained, and dependents
// cannot launch before every CTA of this grid has started.  The epilogue's global inputs
// (EPI_RESID: residual x; EPI_QKV: the RoPE cos / sin rows of each column's position) are
// bulk-copied into shared memory while the mainloop runs, so the fused epilogue loop never
// waits on a global load (it was latency-bound on them at N = 256: 20 us for QKV).
namespace dec {
template <int BN>
struct Cfg {
  static constexpr int HB = BN / 2;                 // activation rows per CTA
  static constexpr int A_BYTES = 128 * kBK * 2;     // 16 KB
  static constexpr int B_BYTES = HB * kBK * 2;
  static constexpr int STAGE = A_BYTES + B_BYTES;
  static constexpr int WMAX = BN / 2;               // widest owned column slice (S >= 2, 16-col grain)
  static constexpr int CTL = 256;
  static constexpr int META = 3 * BN * 4;
  static constexpr int RED = 2 * 4 * BN * 4;
  static constexpr int FIXED = 1024 + CTL + META + RED;
  static constexpr int FIT = (227 * 1024 - FIXED) / STAGE;
  static constexpr int STAGES = FIT > 8 ? 8 : FIT;
  static constexpr int RING = STAGES * STAGE;
  static constexpr int SMEM = FIXED + RING;
  static_assert(STAGES >= 4, "decode pair ring depth");
};
// after the mainloop the ring holds the S - 1 received slices (slot 0 then the summed slice)
// and the epilogue inputs (128 floats per owned column)
template <int BN>
__host__ __device__ inline bool dec_fits(int S, int wslot) {
  return (int64_t)S * wslot * 512 + 16384 <= Cfg<BN>::RING;  // + the EPI_QKV staging of 2 groups
}
// owned columns of pair p: 16-column chunks split as evenly as possible; a workspace slot
// holds the widest slice (dec_slot columns of 128 fp32)
__host__ __device__ inline int dec_col(int BN, int S, int p) { return 16 * ((BN / 16) * p / S); }
__host__ __device__ inline int dec_slot(int BN, int S) { return 16 * ((BN / 16 + S - 1) / S); }
constexpr int kDecPf = 8;  // weight k-blocks prefetched into L2 beyond the ring
RT_DEV void st_release_gpu(unsigned* p, unsigned v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
RT_DEV unsigned ld_acquire_gpu(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
}  // namespace dec

template <int BN, int MODE>
__global__ void __launch_bounds__(kDecThreads, 1)
    k_gemm_dec(const __grid_constant__ TmaMap tmA, const __grid_constant__ TmaMap tmB, GemmArgs g, int S,
               float* ws, unsigned* flags, unsigned epoch) {
  using C = dec::Cfg<BN>;
  constexpr int STAGES = C::STAGES;
  extern __shared__ unsigned char smem_raw[];
  unsigned char* smem = (unsigned char*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  unsigned char* sA = smem;
  unsigned char* sB = smem + STAGES * C::A_BYTES;
  unsigned char* ctl = smem + C::RING;
  uint64_t* full = reinterpret_cast<uint64_t*>(ctl);
  uint64_t* empty = full + STAGES;
  uint64_t* done = empty + STAGES;
  uint64_t* pf_bar = done + 1;
  uint64_t* rx_bar = pf_bar + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(rx_bar + 1);
  EpiSmem sm;
  sm.pos = reinterpret_cast<int*>(ctl + C::CTL);
  sm.page = sm.pos + BN;
  sm.inv = reinterpret_cast<float*>(sm.page + BN);
  sm.redv = reinterpret_cast<float*>(ctl + C::CTL + C::META);
  sm.redi = reinterpret_cast<int*>(sm.redv + 4 * BN);
  sm.bn = BN;
  __shared__ long long s_mark[9];
  sm.mark = s_mark;

  TraceScope tr(TK_GEMM | ((uint32_t)MODE << 8) | ((uint32_t)(2 * S) << 16));
  __shared__ unsigned long long s_tdone;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int h = (int)cluster_rank();                // CTA of the pair
  const int pr = (int)blockIdx.x >> 1;              // pair index in the grid
  const int t = pr / S, p = pr - (pr / S) * S;      // pair-tile, split
  const int m_tile = 2 * t + h;
  const int kbt = g.kb_total;
  const int kb0 = (kbt * p) / S, kb1 = (kbt * (p + 1)) / S;
  const int cb = dec::dec_col(BN, S, p), ce = dec::dec_col(BN, S, p + 1);
  const int wslot = dec::dec_slot(BN, S);
  // workspace: slot (tile, half, owner q, source p) of wslot columns x 128 rows
  auto slot_ptr = [&](int q, int src) {
    return ws + ((((size_t)t * 2 + h) * S + q) * S + src) * (size_t)wslot * 128;
  };
  float* xp = reinterpret_cast<float*>(smem) + (size_t)(S - 1) * wslot * 128;  // epilogue inputs (ring)
  sm.xp = xp;
  sm.xp_sin = wslot * 64;
  sm.stg = MODE == EPI_QKV ? reinterpret_cast<bf16*>(xp + (size_t)wslot * 128) : nullptr;  // 8 KB (ring)

  if (warp == 0 && lane == 0) {
    prefetch_tmap(&tmA);
    prefetch_tmap(&tmB);
    for (int i = 0; i < STAGES; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    mbar_init(done, 1);
    mbar_init(pf_bar, 1);
    mbar_init(rx_bar, 1);
    fence_mbar_init();
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(BN));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  cluster_arrive();  // both CTAs' barriers are initialised before anyone signals them
  cluster_wait();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  constexpr bool QKV_LIKE = MODE == EPI_QKV || MODE == EPI_PART;
  constexpr bool PART = MODE == EPI_PART;  // raw partials, no split-K exchange
  if (!QKV_LIKE && threadIdx.x == 0) pdl_trigger();

  if (warp == 0) {
    if (lane == 0) {
      const uint32_t full0 = dsmem_addr(smem_u32(full), 0);  // the pair leader's full barriers
      const uint32_t bytes = 2u * C::STAGE;
      const int pre_k = min(STAGES, kb1 - kb0);
      // weights do not depend on the previous kernel: the first stages before its completion
      for (int i = 0; i < pre_k; ++i) {
        if (h == 0) mbar_arrive_expect_tx(&full[i], bytes);
        tma_load_2d_pair(sA + i * C::A_BYTES, &tmA, 0, (m_tile * kbt + kb0 + i) * 128, full0 + i * 8);
      }
      pdl_wait();
      if (QKV_LIKE) pdl_trigger();
      tr.ready();
      for (int i = 0; i < pre_k; ++i)
        tma_load_2d_pair(sB + i * C::B_BYTES, &tmB, (kb0 + i) * kBK, h * C::HB, full0 + i * 8);
      // weight k-blocks beyond the ring go to L2 ahead of time (cp.async.bulk.prefetch.L2): the
      // ring alone keeps ~64 KB of HBM reads in flight per SM (B comes from L2), ~4.3 TB/s
      // over 128 SMs at the loaded HBM latency; the prefetch distance adds kDecPf k-blocks
      const bf16* wt = g.w + ((size_t)m_tile * kbt + kb0) * (128 * kBK);
      const int n_kb = kb1 - kb0;
      for (int i = pre_k; i < min(n_kb, pre_k + dec::kDecPf); ++i)
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(wt + (size_t)i * (128 * kBK)),
                     "r"((uint32_t)C::A_BYTES)
                     : "memory");
      for (int i = pre_k; i < n_kb; ++i) {
        const int st = i % STAGES;
        mbar_wait(&empty[st], (uint32_t)(((i / STAGES) & 1) ^ 1));
        if (h == 0) mbar_arrive_expect_tx(&full[st], bytes);
        tma_load_2d_pair(sA + st * C::A_BYTES, &tmA, 0, (m_tile * kbt + kb0 + i) * 128, full0 + st * 8);
        tma_load_2d_pair(sB + st * C::B_BYTES, &tmB, (kb0 + i) * kBK, h * C::HB, full0 + st * 8);
        if (i + dec::kDecPf < n_kb)
          asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(wt + (size_t)(i + dec::kDecPf) * (128 * kBK)),
                       "r"((uint32_t)C::A_BYTES)
                       : "memory");
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    if (h == 0 && lane == 0) {
      constexpr uint32_t idesc = umma_idesc(256, BN);
      for (int i = 0; i < kb1 - kb0; ++i) {
        const int st = i % STAGES;
        mbar_wait(&full[st], (uint32_t)((i / STAGES) & 1));
        tc_fence_after();
        const uint32_t a0 = smem_u32(sA + st * C::A_BYTES);
        const uint32_t b0 = smem_u32(sB + st * C::B_BYTES);
#pragma unroll
        for (int k = 0; k < kBK / 16; ++k)
          umma_f16_pair(tmem, umma_desc_sw128(a0 + k * 32), umma_desc_sw128(b0 + k * 32), idesc,
                        (i > 0 || k > 0) ? 1u : 0u);
        umma_commit_pair(&empty[st], 0x3);
      }
      umma_commit_pair(done, 0x3);
    }
    __syncwarp();
  } else {
    // two epilogue groups of 4 warps (warps 2-5, 6-9): both cover the 128 TMEM lanes (lane
    // quarter = warp % 4) and split the columns, so the latency-bound exchange, sum and fused
    // loops run on 8 warps (2 per SM sub-partition)
    pdl_wait();
    const int grp = (warp - 2) >> 2;
    const int et = (warp & 3) * 32 + lane;
    const uint32_t tb = tmem + ((uint32_t)((warp & 3) * 32) << 16);
    // owned columns of this group: 16-column halves of [cb, ce)
    const int gm = cb + 16 * ((((ce - cb) >> 4) + 1) >> 1);
    const int gcb = grp == 0 ? cb : gm, gce = grp == 0 ? gm : ce;
    EpiSmem gs = sm;
    gs.bar = 1 + grp;
    gs.mark = grp == 0 ? s_mark : nullptr;
    // per-column metadata of the owned columns while the mainloop runs (group 0; ordered
    // before group 1's reads by the 256-thread barrier after the exchange writes)
    if (grp == 0) column_meta<MODE>(g, sm, m_tile, 0, cb, ce, et, false);
    mbar_wait(done, 0);
    tc_fence_after();
    if (et == 0 && grp == 0) {
      s_tdone = gtimer();
      const long long c0 = clock64();
#pragma unroll
      for (int i = 0; i < 9; ++i) s_mark[i] = c0;
    }
    if constexpr (PART) {  // raw partial of split p -> part[p][n][m]; group g: columns [g BN/2, ..)
      const int m = m_tile * 128 + et;
      float* dst = g.part + (size_t)p * g.part_ld_n * g.M + m;
      const int c_hi = min((grp + 1) * (BN / 2), g.N);
#pragma unroll 1
      for (int c0 = grp * (BN / 2); c0 < c_hi; c0 += 16) {
        float v[16];
        tmem_ld16(tb + (uint32_t)c0, v);
#pragma unroll
        for (int j = 0; j < 16; ++j)
          if (c0 + j < c_hi) __stcg(dst + (size_t)(c0 + j) * g.M, v[j]);
      }
    } else {
    // the ring is free: the epilogue inputs -> shared memory (bulk copies on pf_bar, one column
    // per thread: issued serially by one thread they took ~10 us for 96 columns), in flight
    // while the split-K exchange runs.  (complete_tx may precede the expect_tx of the phase.)
    if (grp == 0) {
      const int cn = min(ce, g.N) - cb;  // owned columns that hold rows
      if constexpr (MODE == EPI_RESID) {
        if (et == 0) mbar_arrive_expect_tx(pf_bar, (uint32_t)max(cn, 0) * 512);
        if (et < cn) bulk_g2s(xp + et * 128, g.x + (size_t)(cb + et) * g.M + m_tile * 128, 512, pf_bar);
      } else if constexpr (MODE == EPI_QKV) {
        const int half = g.qkv.hd >> 1;
        const uint32_t rb = (uint32_t)half * 4;
        if (et == 0) mbar_arrive_expect_tx(pf_bar, (uint32_t)max(cn, 0) * 2 * rb);
        if (et < cn) {
          const int pos = sm.pos[cb + et];
          bulk_g2s(xp + et * 64, g.qkv.cos + (size_t)pos * half, rb, pf_bar);
          bulk_g2s(xp + sm.xp_sin + et * 64, g.qkv.sin + (size_t)pos * half, rb, pf_bar);
        }
      } else {
        if (et == 0) mbar_arrive(pf_bar);
      }
    }
    // ---- split-K exchange through L2: the slices other pairs own -> their workspace slots
    // (16-column chunks alternate between the groups)
    for (int q = 0, j = 0; q < S; ++q) {
      if (q == p) continue;
      const int qb = dec::dec_col(BN, S, q), qe = dec::dec_col(BN, S, q + 1);
      float* dst = slot_ptr(q, p) + et;
#pragma unroll 1
      for (int c0 = qb; c0 < qe; c0 += 16, ++j) {
        if ((j & 1) != grp) continue;
        float v[16];
        tmem_ld16(tb + (uint32_t)c0, v);
#pragma unroll
        for (int jj = 0; jj < 16; ++jj) __stcg(dst + (size_t)(c0 - qb + jj) * 128, v[jj]);
      }
    }
    if (et == 0 && grp == 0) s_mark[1] = clock64();  // (trace marks: group 0 only)
    asm volatile("bar.sync 3, 256;" ::: "memory");  // every row of this CTA's slices is written
    unsigned* myflags = flags + ((size_t)t * 2 + h) * S;
    if (et == 0 && grp == 0) {
      __threadfence();
      dec::st_release_gpu(myflags + p, epoch);
    }
    if (et == 0 && grp == 0) s_mark[2] = clock64();
    // wait for the S - 1 contributors of my slice, then bulk-copy their slices (ring slots
    // j = 0 .. S - 2 in pair order, wslot columns each) into shared memory at once
    float* R = reinterpret_cast<float*>(smem);
    const uint32_t slice_bytes = (uint32_t)(ce - cb) * 512;
    if (et == 0 && grp == 0) {
      for (int q = 0; q < S; ++q)
        if (q != p)
          while (dec::ld_acquire_gpu(myflags + q) != epoch) __nanosleep(32);
      asm volatile("fence.proxy.async.global;" ::: "memory");  // generic writes -> bulk-copy reads
      mbar_arrive_expect_tx(rx_bar, (uint32_t)(S - 1) * slice_bytes);
      for (int q = 0, j = 0; q < S; ++q)
        if (q != p) bulk_g2s(R + (size_t)(j++) * wslot * 128, slot_ptr(p, q), slice_bytes, rx_bar);
    }
    if (et == 0 && grp == 0) s_mark[3] = clock64();
    mbar_wait(rx_bar, 0);
    // ---- sum the S partials of the group's columns in pair order (deterministic) -> T (= slot
    // 0: every element is read, then written, by the same thread)
    float* T = R;
#pragma unroll 1
    for (int c0 = gcb; c0 < gce; c0 += 16) {
      float own[16], acc[16];
      tmem_ld16(tb + (uint32_t)c0, own);
#pragma unroll
      for (int j = 0; j < 16; ++j) acc[j] = 0.f;
      for (int q = 0, jq = 0; q < S; ++q) {
        if (q == p) {
#pragma unroll
          for (int j = 0; j < 16; ++j) acc[j] += own[j];
        } else {
          const float* src = R + (size_t)(jq++) * wslot * 128 + (size_t)(c0 - cb) * 128 + et;
#pragma unroll
          for (int j = 0; j < 16; ++j) acc[j] += (c0 + j < gce) ? src[j * 128] : 0.f;
        }
      }
#pragma unroll
      for (int j = 0; j < 16; ++j)
        if (c0 + j < gce) T[(c0 - cb + j) * 128 + et] = acc[j];
    }
    mbar_wait(pf_bar, 0);  // prefetched epilogue inputs
    epi_bar(gs.bar);
    // the group's view of the prefetched inputs (indexed from its first column) and staging
    gs.xp = xp + (size_t)(gcb - cb) * (MODE == EPI_QKV ? 64 : 128);
    if (gs.stg) gs.stg = sm.stg + grp * (2 * kEpiCh * 128);
    const TileSrc ts{T - (size_t)cb * 128, nullptr, 0u, 1, 0, BN, 0, 0};
    if (gcb < gce) epilogue<MODE>(g, gs, ts, m_tile, 0, gcb, gce, et, true);
    }  // !PART
    if (et == 0 && grp == 0) s_mark[8] = clock64();
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x == 0) {
    tr.aux(s_tdone);
    auto dd = [&](int i) {
      const long long d = s_mark[i + 1] - s_mark[i];
      return (unsigned long long)(uint32_t)(d > 0 ? d : 0);
    };
    trace_phase(TK_PHASE | TK_GEMM | ((uint32_t)MODE << 8) | ((uint32_t)(2 * S) << 16), dd(0) | (dd(1) << 32),
                dd(2) | (dd(3) << 32), dd(4) | (dd(5) << 32), dd(6) | (dd(7) << 32));
  }
  cluster_arrive();  // no CTA deallocates while its pair peer may still use the shared TMEM pair state
  cluster_wait();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(BN));
  }
}

// ------------------------------------------------------------- host side
static PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = (PFN_cuTensorMapEncodeTiled_v12000)p;
  }
  return fn;
}

static bool make_tma_2d_bf16_sw(TmaMap* out, const void* base, uint64_t inner, uint64_t rows, uint32_t box_inner,
                                uint32_t box_rows, CUtensorMapSwizzle sw) {
  auto enc = get_encode();
  if (!enc) return false;
  cuuint64_t dims[2] = {inner, rows};
  cuuint64_t strides[1] = {inner * 2};
  cuuint32_t box[2] = {box_inner, box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(reinterpret_cast<CUtensorMap*>(out->bytes), CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2,
                   const_cast<void*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, sw,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

bool make_tma_2d_bf16(TmaMap* out, const void* base, uint64_t inner, uint64_t rows, uint32_t box_inner,
                      uint32_t box_rows) {
  auto enc = get_encode();
  if (!enc) return false;
  cuuint64_t dims[2] = {inner, rows};
  cuuint64_t strides[1] = {inner * 2};
  cuuint32_t box[2] = {box_inner, box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(reinterpret_cast<CUtensorMap*>(out->bytes), CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2,
                   const_cast<void*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

bool make_gemm_act_maps(GemmTmaSet* out, const void* base, int K, int rows_cap) {
  out->rows_cap = rows_cap;
  return make_tma_2d_bf16(&out->m32, base, K, rows_cap, kBK, 32) &&
         make_tma_2d_bf16(&out->m64, base, K, rows_cap, kBK, 64) &&
         make_tma_2d_bf16(&out->m80, base, K, rows_cap, kBK, 80) &&
         make_tma_2d_bf16(&out->m96, base, K, rows_cap, kBK, 96) &&
         make_tma_2d_bf16(&out->m128, base, K, rows_cap, kBK, 128) &&
         make_tma_2d_bf16(&out->m160, base, K, rows_cap, kBK, 160) &&
         make_tma_2d_bf16(&out->m192, base, K, rows_cap, kBK, 192) &&
         make_tma_2d_bf16(&out->m256, base, K, rows_cap, kBK, 256);
}

// Kernel choice for N activation rows: the N tile (UMMA N) and, above 128 rows, whether the
// CTA-pair kernel runs (when eligible, see launch_gemm_epi).  Up to 128 rows the powers of
// two (decode, single SM).  Above: for the model's projection shapes the measured table
// gemm_policy.inc (tools/gemm_policy_tune.py: every candidate of a 32-row bucket timed back to
// back; vs the rule below 11-18 % less time summed over 160..4096 rows); otherwise the width
// among {160, 192, 256} with the least padded MMA work (n-tiles x BN), then fewer n-tiles
// (a padded column costs a full MMA column), with the pair kernel at 192 / 256.
// Overrides (parity tests, the tuner): GemmArgs::force_bn / force_path.
#include "gemm_policy.inc"
struct GemmChoice {
  int bn;
  bool pair;
};
static GemmChoice gemm_choice(int M, int K, int N, int force_bn = 0, int force_path = GEMM_PATH_AUTO) {
  GemmChoice c{256, false};
  if (N <= 32) c = {32, false};
  else if (N <= 64) c = {64, false};
  else if (N <= 128) c = {128, false};
  else {
    bool found = false;
    for (const GemmPolicyRow& r : kGemmPolicy)
      if (r.M == M && r.K == K && N <= r.n_max) {
        const int code = r.code[(N - 129) / 32] - '0';
        c.bn = code % 3 == 0 ? 160 : (code % 3 == 1 ? 192 : 256);
        c.pair = code >= 3;
        found = true;
        break;
      }
    if (!found) {
      int best_t = INT_MAX;
      long long best_w = LLONG_MAX;
      for (int bn : {160, 192, 256}) {
        const int t = (N + bn - 1) / bn;
        const long long w = (long long)t * bn;
        if (w < best_w || (w == best_w && t < best_t)) {
          c.bn = bn;
          best_w = w;
          best_t = t;
        }
      }
      c.pair = c.bn >= 192;
    }
  }
  if (force_bn > 0) c.bn = force_bn;
  if (force_path != GEMM_PATH_AUTO) c.pair = force_path == GEMM_PATH_PAIR;
  return c;
}
int gemm_bn(int M, int K, int N) { return gemm_choice(M, K, N).bn; }

template <int BN, int MODE>
static void ensure_attrs() {
  using C = GemmCfg<BN>;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_gemm_tc<BN, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
    cudaFuncSetAttribute(k_gemm_tc<BN, MODE>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    attr = true;
  }
}

// Cluster split count (measured on B200, tools/gemm_bench.py, N = 64): a split-K cluster
// only pays off while every cluster is co-resident in ONE wave; with >= 148 tiles plain
// tiles (S = 1) already cover the SMs.  Measured co-residency of 2-CTA/SM clusters holds
// up to 256 CTAs (O / down: 32 x 8 = 256 -> 11.7 / 26 us) but not 288 (QKV 48 x 6:
// 12 -> 19 us, 32 x 9: 11 -> 19 us), so S = max{S <= 8 : tiles x S <= 256, >= 4 k-blocks
// per CTA} (cudaOccupancyMaxActiveClusters under-reports and is only a cap).
int gemm_choose_splits(int M, int N, int K) {
  const int bn = gemm_bn(M, K, N);
  const int tiles = ((M + 127) / 128) * ((N + bn - 1) / bn);
  const int kb = K / kBK;
  if (tiles >= 148) return 1;
  const int budget = bn <= 128 ? 256 : 128;
  int best = 1;
  for (int s = 2; s <= 8 && kb / s >= 4; ++s)
    if (tiles * s <= budget) best = s;
  return best;
}

template <int BN, int MODE>
static cudaError_t launch_bn(const TmaMap& b, const GemmArgs& g, int S, cudaStream_t s) {
  using C = GemmCfg<BN>;
  ensure_attrs<BN, MODE>();
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(S, g.tile_count, 1);
  cfg.blockDim = dim3(kGemmThreads);
  cfg.dynamicSmemBytes = C::SMEM;
  cfg.stream = s;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  at[1].id = cudaLaunchAttributeClusterDimension;
  at[1].val.clusterDim.x = S;
  at[1].val.clusterDim.y = 1;
  at[1].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 2;
  return cudaLaunchKernelEx(&cfg, k_gemm_tc<BN, MODE>, b, g);
}

template <int MODE>
static cudaError_t launch_mode(const GemmTmaSet& x, const GemmArgs& g, int bn, int S, cudaStream_t s) {
  if (bn == 32) return launch_bn<32, MODE>(x.m32, g, S, s);
  if (bn == 64) return launch_bn<64, MODE>(x.m64, g, S, s);
  if (bn == 128) return launch_bn<128, MODE>(x.m128, g, S, s);
  if (bn == 160) return launch_bn<160, MODE>(x.m160, g, S, s);
  if (bn == 192) return launch_bn<192, MODE>(x.m192, g, S, s);
  return launch_bn<256, MODE>(x.m256, g, S, s);
}

static int sm_count() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

template <int BN, int MODE>
static cudaError_t launch_sk_bn(const TmaMap& b, const GemmArgs& g, const SkArgs& a, cudaStream_t s) {
  using C = sk::Cfg<BN>;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_gemm_sk<BN, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
    attr = true;
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(a.P);
  cfg.blockDim = dim3(kGemmThreads);
  cfg.dynamicSmemBytes = C::SMEM;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, k_gemm_sk<BN, MODE>, b, g, a);
}
template <int MODE>
static cudaError_t launch_sk_mode(const GemmTmaSet& x, const GemmArgs& g, const SkArgs& a, int bn, cudaStream_t s) {
  if (bn == 160) return launch_sk_bn<160, MODE>(x.m160, g, a, s);
  if (bn == 192) return launch_sk_bn<192, MODE>(x.m192, g, a, s);
  return launch_sk_bn<256, MODE>(x.m256, g, a, s);
}

// ---- CTA-pair launch (k_gemm_2sm)
// weight operand of the pair kernel: the pre-tiled image read as rows of 64 bf16 (128 B), one
// 16 KB box per (m-tile, k-block); the map depends only on (pointer, rows): cached
static const TmaMap* weight_map(const bf16* w, uint64_t rows) {
  static std::map<std::pair<const void*, uint64_t>, TmaMap> cache;  // node-based: pointers stay valid
  static std::mutex mu;  // engines may run on different host threads
  std::lock_guard<std::mutex> lock(mu);
  const auto key = std::make_pair((const void*)w, rows);
  auto it = cache.find(key);
  if (it != cache.end()) return &it->second;
  TmaMap m;
  if (!make_tma_2d_bf16_sw(&m, w, kBK, rows, kBK, 128, CU_TENSOR_MAP_SWIZZLE_NONE)) return nullptr;
  return &cache.emplace(key, m).first->second;
}
template <int BN, int MODE>
static cudaError_t launch_2sm_bn(const TmaMap& am, const TmaMap& bm, const TmaMap& bms, const GemmArgs& g, int PT,
                                 SkArgs a, cudaStream_t s) {
  using C = sm2::Cfg<BN>;
  static int slots = 0;
  if (PT <= 0) {  // query: co-resident pairs
    if (slots) return cudaSuccess;
  }
  cudaLaunchConfig_t cfg{};
  cfg.blockDim = dim3(kDecThreads);
  cfg.dynamicSmemBytes = C::SMEM;
  cfg.stream = s;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = 2;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[1].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  cfg.attrs = at;
  if (!slots) {  // co-resident CTA pairs (persistent grid)
    cudaFuncSetAttribute(k_gemm_2sm<BN, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
    cfg.gridDim = dim3(sm_count() & ~1);
    cfg.numAttrs = 1;
    int n = 0;
    if (cudaOccupancyMaxActiveClusters(&n, k_gemm_2sm<BN, MODE>, &cfg) != cudaSuccess || n <= 0) {
      cudaGetLastError();
      n = sm_count() / 2;
    }
    slots = n;
  }
  if (PT <= 0) return cudaSuccess;
  const int n_pairs = std::min(PT, slots);
  a.P = n_pairs;
  a.head = PT;
  a.sub_s = 0;
  // partial last round of whole pair-tiles: if its sub-tiles fit one per pair, run them
  // instead (gate/up at 384 / 512 rows: 224 pair-tiles = 3 x 74 + 2 -> 2 x 3 / 2 x 4 sub-tiles)
  if (PT > n_pairs && PT % n_pairs && BN % kPairSubW == 0 &&
      (PT % n_pairs) * (BN / kPairSubW) <= n_pairs) {
    a.head = PT - PT % n_pairs;
    a.sub_s = BN / kPairSubW;
  }
  cfg.gridDim = dim3(2 * n_pairs);
  cfg.numAttrs = 2;
  return cudaLaunchKernelEx(&cfg, k_gemm_2sm<BN, MODE>, am, bm, bms, g, a);
}
template <int MODE>
static cudaError_t launch_2sm_mode(const TmaMap& am, const GemmTmaSet& x, const GemmArgs& g, int bn, int PT,
                                   const SkArgs& a, cudaStream_t s) {
  if (bn == 128) return launch_2sm_bn<128, MODE>(am, x.m64, x.m32, g, PT, a, s);
  if (bn == 160) return launch_2sm_bn<160, MODE>(am, x.m80, x.m32, g, PT, a, s);
  if (bn == 192) return launch_2sm_bn<192, MODE>(am, x.m96, x.m32, g, PT, a, s);
  return launch_2sm_bn<256, MODE>(am, x.m128, x.m32, g, PT, a, s);
}
// (pairs at 160-wide tiles only where the table measured them faster: their rounds quantise
// worse than the single-SM stream-K kernel, e.g. gate/up 83.3 -> 88.5 us at 320 rows)
// co-resident CTA pairs of the pair kernel at this tile width (occupancy query, cached)
template <int BN>
static int pair_slots_bn() {
  static int n = 0;
  if (!n) {
    GemmArgs g{};
    TmaMap t{};
    launch_2sm_bn<BN, EPI_STORE>(t, t, t, g, 0, SkArgs{}, nullptr);
    cudaLaunchConfig_t cfg{};
    cfg.blockDim = dim3(kDecThreads);
    cfg.dynamicSmemBytes = sm2::Cfg<BN>::SMEM;
    cfg.gridDim = dim3(sm_count() & ~1);
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 2;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    if (cudaOccupancyMaxActiveClusters(&n, k_gemm_2sm<BN, EPI_STORE>, &cfg) != cudaSuccess || n <= 0) {
      cudaGetLastError();
      n = sm_count() / 2;
    }
  }
  return n;
}
static int pair_slots(int bn) {
  return bn == 160 ? pair_slots_bn<160>() : (bn == 192 ? pair_slots_bn<192>() : pair_slots_bn<256>());
}


// ---- decode CTA-pair split-K launch (k_gemm_dec)
template <int BN, int MODE>
static cudaError_t launch_dec_bn(const TmaMap& am, const TmaMap& bm, const GemmArgs& g, int PT, int S,
                                 cudaStream_t s) {
  using C = dec::Cfg<BN>;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_gemm_dec<BN, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
    attr = true;
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(2 * S * PT);
  cfg.blockDim = dim3(kDecThreads);
  cfg.dynamicSmemBytes = C::SMEM;
  cfg.stream = s;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = 2;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[1].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  cfg.attrs = at;
  cfg.numAttrs = 2;
  return cudaLaunchKernelEx(&cfg, k_gemm_dec<BN, MODE>, am, bm, g, S, g.dec_ws, g.dec_flags, g.dec_epoch);
}
template <int MODE>
static cudaError_t launch_dec_mode(const TmaMap& am, const GemmTmaSet& x, const GemmArgs& g, int bn, int PT, int S,
                                   cudaStream_t s) {
  if (bn == 64) return launch_dec_bn<64, MODE>(am, x.m32, g, PT, S, s);
  if (bn == 128) return launch_dec_bn<128, MODE>(am, x.m64, g, PT, S, s);
  return launch_dec_bn<256, MODE>(am, x.m128, g, PT, S, s);
}
// split count of the decode pair kernel: S x pair-tiles <= the SM pairs (one CTA per SM, every
// pair resident at once: the owners spin on their contributors), >= 4 k-blocks per pair
static int dec_splits(int PT, int kbt, int bn) {
  const int pairs = sm_count() / 2;
  int best = 0;
  for (int S = 2; S <= 8; ++S) {
    const int w = dec::dec_slot(bn, S);
    const bool fits = bn == 64 ? dec::dec_fits<64>(S, w) : (bn == 128 ? dec::dec_fits<128>(S, w) : dec::dec_fits<256>(S, w));
    if (fits && PT * S <= pairs && kbt / S >= 4) best = S;
  }
  return best;
}
int64_t gemm_dec_ws_floats(int M, int N, int K) {
  const int PT = (M + 127) / 256;
  const int bn = N <= 64 ? 64 : (N <= 128 ? 128 : 256);
  const int S = dec_splits(PT, K / kBK, bn);
  return S < 2 ? 0 : (int64_t)PT * 2 * S * S * dec::dec_slot(bn, S) * 128;
}
// launch the decode pair kernel if it applies (returns cudaErrorNotSupported otherwise)
static cudaError_t try_launch_dec(const bf16* w_tiled, const GemmTmaSet& x, GemmArgs g, int force_s,
                                  cudaStream_t s) {
  const int m_tiles = (g.M + 127) / 128;
  const bool part = g.mode == EPI_PART;  // no exchange: no workspace / flags needed
  if (!part && (!g.dec_ws || !g.dec_flags)) return cudaErrorNotSupported;
  if (g.N > 256 || g.N < 1 || g.M % 256 || g.K % kBK || g.mode == EPI_ARGMAX) return cudaErrorNotSupported;
  const int bn = g.N <= 64 ? 64 : (g.N <= 128 ? 128 : 256);
  const int PT = m_tiles / 2;
  const int kbt = g.K / kBK;
  int S = dec_splits(PT, kbt, bn);
  if (force_s >= 2 && force_s <= S) S = force_s;  // op-level override (tools / tests): fewer splits
  if (S < 2) return cudaErrorNotSupported;
  if (!part && ((int64_t)PT * 2 * S * S * dec::dec_slot(bn, S) * 128 > g.dec_ws_floats || PT * 2 * S > g.dec_flags_cap))
    return cudaErrorNotSupported;
  const TmaMap* am = weight_map(w_tiled, (uint64_t)m_tiles * kbt * 128);
  if (!am) return cudaErrorNotSupported;
  g.w = w_tiled;
  g.kb_total = kbt;
  g.m_tiles = m_tiles;
  g.n_tiles = 1;
  g.l2_evict_first = 0;
  switch (g.mode) {
    case EPI_STORE: return launch_dec_mode<EPI_STORE>(*am, x, g, bn, PT, S, s);
    case EPI_QKV: return launch_dec_mode<EPI_QKV>(*am, x, g, bn, PT, S, s);
    case EPI_RESID: return launch_dec_mode<EPI_RESID>(*am, x, g, bn, PT, S, s);
    case EPI_SWIGLU: return launch_dec_mode<EPI_SWIGLU>(*am, x, g, bn, PT, S, s);
    case EPI_PART: return launch_dec_mode<EPI_PART>(*am, x, g, bn, PT, S, s);
    default: return cudaErrorNotSupported;
  }
}

int64_t gemm_sk_ws_floats() { return (int64_t)sm_count() * 2 * 256 * 128; }

// Split count of the decode QKV projection in EPI_PART (QKV folded into the attention):
// the decode pair kernel's at 129..256 rows, the cluster split-K kernel's at <= 128 rows;
// 0 = not supported at this shape (the caller keeps EPI_QKV).  launch_gemm_epi runs exactly
// this choice, so the attention knows how many partials to sum.
int gemm_part_splits(int M, int K, int N) {
  if (N < 1 || N > 256 || K % kBK) return 0;
  if (N > 128) {
    if (M % 256) return 0;
    const int S = dec_splits(M / 256, K / kBK, 256);
    return S >= 2 ? S : 0;
  }
  return std::max(1, std::min(gemm_choose_splits(M, N, K), std::min(16, K / kBK)));
}

cudaError_t launch_gemm_epi(const bf16* w_tiled, const GemmTmaSet& x, GemmArgs g, int splits, cudaStream_t s) {
  if (g.mode == EPI_PART) {  // only the two decode kernels write raw partials
    const int S = gemm_part_splits(g.M, g.K, g.N);
    if (S == 0 || !g.part) return cudaErrorInvalidValue;
    if (g.N > 128) return try_launch_dec(w_tiled, x, g, 0, s);
    g.force_path = GEMM_PATH_SPLITK;
    g.force_bn = 0;
    splits = S;
  }
  // decode rows on the few-tile projections (<= 256 rows, 129..256 by default): CTA pairs with
  // a cluster split-K (k_gemm_dec)
  if (g.force_path == GEMM_PATH_DEC || (g.force_path == GEMM_PATH_AUTO && g.N > 128 && g.N <= 256)) {
    const cudaError_t r = try_launch_dec(w_tiled, x, g, g.force_path == GEMM_PATH_DEC ? splits : 0, s);
    if (r != cudaErrorNotSupported) return r;
  }
  const GemmChoice gc = gemm_choice(g.M, g.K, g.N, g.force_bn, g.force_path);
  const int bn = gc.bn;
  // CTA-pair kernel for the tensor-bound prefill path: every pair busy (at least one
  // pair-tile per co-resident pair) and an even number of 128-row m-tiles
  if (g.N > 128 && g.K % kBK == 0 && gc.pair) {
    const int m_tiles = (g.M + 127) / 128, n_tiles = (g.N + bn - 1) / bn;
    const int PT = (m_tiles / 2) * n_tiles;
    const int slots = pair_slots(bn);
    if (m_tiles % 2 == 0 && (PT >= slots || g.force_path == GEMM_PATH_PAIR)) {
      const TmaMap* am = weight_map(w_tiled, (uint64_t)m_tiles * (g.K / kBK) * 128);
      if (am) {
        g.w = w_tiled;
        g.kb_total = g.K / kBK;
        g.m_tiles = m_tiles;
        g.n_tiles = n_tiles;
        g.l2_evict_first = 0;
        SkArgs a{};
        a.n_tiles = n_tiles;
        switch (g.mode) {
          case EPI_STORE: return launch_2sm_mode<EPI_STORE>(*am, x, g, bn, PT, a, s);
          case EPI_ARGMAX: return launch_2sm_mode<EPI_ARGMAX>(*am, x, g, bn, PT, a, s);
          case EPI_QKV: return launch_2sm_mode<EPI_QKV>(*am, x, g, bn, PT, a, s);
          case EPI_RESID: return launch_2sm_mode<EPI_RESID>(*am, x, g, bn, PT, a, s);
          case EPI_SWIGLU: return launch_2sm_mode<EPI_SWIGLU>(*am, x, g, bn, PT, a, s);
          default: return cudaErrorInvalidValue;
        }
      }
    }
  }
  // hybrid data-parallel + stream-K persistent kernel for the tensor-bound prefill path
  // (N > 128 rows, more than two waves of tiles) when the caller provides its workspace
  if (g.sk_ws && g.sk_cnt && g.N > 128 && g.mode != EPI_ARGMAX && g.K % kBK == 0 &&
      g.force_path != GEMM_PATH_SPLITK) {
    g.w = w_tiled;
    g.kb_total = g.K / kBK;
    g.m_tiles = (g.M + 127) / 128;
    g.l2_evict_first = 0;
    SkArgs a{};
    a.n_tiles = (g.N + bn - 1) / bn;
    const int T = g.m_tiles * a.n_tiles;
    const int P = sm_count();
    const long long I_sk = (long long)(T <= P ? T : (T % P) + P) * g.kb_total;
    // only with a data-parallel part (T > 2 waves): measured faster there (gate/up N = 320 /
    // 384 / 512: 103 / 108 / 122 -> 89 / 95 / 116 us) and slower for all-stream-K shapes
    // (few-tile projections pay multi-contributor fixups; the cluster split-K path is better)
    // (all-stream-K at <= 2 waves is not supported: it measured slower, RT_SK_MODE in round 1,
    // and its fixup schedule assumes the data-parallel waves in front)
    const int min_t = 2 * P + 1;
    a.all_sk = T <= 2 * P ? 1 : 0;
    if (T <= g.sk_cnt_cap && I_sk >= P && T >= min_t) {
      a.P = P;
      a.ws = g.sk_ws;
      a.cnt = g.sk_cnt;
      switch (g.mode) {
        case EPI_STORE: return launch_sk_mode<EPI_STORE>(x, g, a, bn, s);
        case EPI_QKV: return launch_sk_mode<EPI_QKV>(x, g, a, bn, s);
        case EPI_RESID: return launch_sk_mode<EPI_RESID>(x, g, a, bn, s);
        case EPI_SWIGLU: return launch_sk_mode<EPI_SWIGLU>(x, g, a, bn, s);
        default: break;
      }
    }
  }
  g.w = w_tiled;
  // weights are read once per n-tile; with several n-tiles the later ones should hit L2
  const int n_tiles = (g.N + bn - 1) / bn;
  g.l2_evict_first = (l2_hint_enabled() && n_tiles == 1) ? 1 : 0;
  g.kb_total = g.K / kBK;
  g.m_tiles = (g.M + 127) / 128;
  g.n_tiles = n_tiles;
  const int tiles = g.m_tiles * n_tiles;
  const bool auto_split = splits <= 0;
  if (splits <= 0) splits = gemm_choose_splits(g.M, g.N, g.K);
  splits = std::max(1, std::min(splits, std::min(16, g.kb_total)));
  auto launch = [&](int tile0, int count, int S) -> cudaError_t {
    g.tile0 = tile0;
    g.tile_count = count;
    switch (g.mode) {
      case EPI_STORE: return launch_mode<EPI_STORE>(x, g, bn, S, s);
      case EPI_ARGMAX: return launch_mode<EPI_ARGMAX>(x, g, bn, S, s);
      case EPI_QKV: return launch_mode<EPI_QKV>(x, g, bn, S, s);
      case EPI_RESID: return launch_mode<EPI_RESID>(x, g, bn, S, s);
      case EPI_SWIGLU: return launch_mode<EPI_SWIGLU>(x, g, bn, S, s);
      case EPI_PART: return launch_mode<EPI_PART>(x, g, bn, S, s);
      default: return cudaErrorInvalidValue;
    }
  };
  // Wave-quantisation tail split (prefill rows, N > 64: tensor-bound, one tile per SM-slot):
  // the full waves of whole tiles in one launch, the remaining tiles in a second launch with
  // a cluster split-K wide enough to spread them over all SMs (gate/up at N = 256: 224 tiles =
  // 148 + 76 -> the 76 tail tiles run as 2-CTA clusters instead of a half-empty second wave)
  const int P = sm_count() * (bn <= 128 ? 2 : 1);  // co-resident CTA slots
  if (auto_split && splits == 1 && bn >= 128 && g.mode != EPI_ARGMAX && tiles > P && tiles % P) {
    const int head = (tiles / P) * P, tail = tiles - head;
    // S = the largest split that still fits the tail into one wave of the slots (a wider split
    // that spills into another wave measured slower: the cluster reduction of 96-128 KB
    // partials costs more than the balance gains, tools/gemm_sweep_n.py)
    const int st = std::min(std::min(16, g.kb_total / 4), std::max(1, P / tail));
    if (st > 1) {
      cudaError_t r = launch(0, head, 1);
      if (r != cudaSuccess) return r;
      return launch(head, tail, st);
    }
  }
  return launch(0, tiles, splits);
}

RT_TRACE_BINDER(trace_bind_gemm)

}  // namespace rt
