// common.cuh — device helpers shared by the sm_100a kernels of the engine.
#pragma once
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <stdint.h>
#include <utility>
#include <stdlib.h>

#define RT_DEV __device__ __forceinline__

typedef __nv_bfloat16 bf16;

// ---------------------------------------------------------------- bf16 helpers
RT_DEV float bf16_lo(uint32_t v) { return __uint_as_float(v << 16); }
RT_DEV float bf16_hi(uint32_t v) { return __uint_as_float(v & 0xFFFF0000u); }
RT_DEV uint16_t f32_to_bf16_bits(float f) {  // RNE (finite inputs)
  return __bfloat16_as_ushort(__float2bfloat16_rn(f));
}
RT_DEV uint32_t pack_bf16x2(float lo, float hi) {
  return (uint32_t)f32_to_bf16_bits(lo) | ((uint32_t)f32_to_bf16_bits(hi) << 16);
}
RT_DEV float bf16_round(float f) { return __bfloat162float(__float2bfloat16_rn(f)); }

// ------------------------------------------------------------- warp utilities
RT_DEV float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
RT_DEV float warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// ------------------------------------------- programmatic dependent launch (PDL)
// Kernels launched with launch_pdl may start while the previous kernel of the stream
// is finishing; they must execute pdl_wait() before touching its outputs.
RT_DEV void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
RT_DEV void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

// RT_NO_PDL=1 disables programmatic dependent launch (A/B measurements)
inline bool pdl_enabled() {
  static const bool on = getenv("RT_NO_PDL") == nullptr;
  return on;
}

// RT_NO_L2HINT=1 disables the evict_first L2 policy on streamed weights / KV (A/B)
inline bool l2_hint_enabled() {
  static const bool on = getenv("RT_NO_L2HINT") == nullptr;
  return on;
}

template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                              Args&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

// ------------------------------------------------ device trace (RT_FLAG_TRACE)
// One record per CTA: %gridid identifies the launch, %globaltimer stamps kernel entry,
// the end of its dependency wait (pdl_wait) and exit — the real in-pipeline timeline
// with PDL overlap, which neither CUDA events (they serialise) nor ncu (it replays)
// can show.  Thread 0 of every CTA writes; off (rec == nullptr) it costs one load.
// t_aux: a kernel-specific phase mark (GEMM: accumulator complete; 0 = none).
// Layout must match rt_trace_rec in rt.h (48 bytes).
struct TraceRec {
  unsigned long long grid;
  uint32_t kind, smid;
  unsigned long long t_entry, t_ready, t_aux, t_exit;
};
struct TraceBuf {
  TraceRec* rec;
  unsigned* n;
  unsigned cap;
};
static __device__ TraceBuf g_trace;  // per translation unit, bound by trace_bind_<tu>()

enum TraceKind : uint32_t {
  TK_GEMM = 1, TK_ATTN = 2, TK_NORM = 3, TK_EMBED = 4, TK_SCHED_PRE = 5, TK_SCHED_POST = 6,
  TK_GATHER = 7, TK_ARGMAX = 8, TK_MERGE = 9, TK_ATTN_PREFILL = 10, TK_RESID = 11, TK_PHASE = 0x80
};

RT_DEV unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
struct TraceScope {
  unsigned long long t0 = 0, t1 = 0, t2 = 0;
  uint32_t kind;
  __device__ explicit TraceScope(uint32_t k) : kind(k) {
    if (threadIdx.x == 0 && g_trace.rec) t0 = t1 = gtimer();
  }
  __device__ void ready() {
    if (threadIdx.x == 0 && g_trace.rec) t1 = gtimer();
  }
  __device__ void aux(unsigned long long t) { t2 = t; }  // thread 0 only
  __device__ ~TraceScope() {
    if (threadIdx.x != 0 || !g_trace.rec) return;
    const unsigned i = atomicAdd(g_trace.n, 1u);
    if (i >= g_trace.cap) return;
    TraceRec r;
    asm volatile("mov.u64 %0, %%gridid;" : "=l"(r.grid));
    asm volatile("mov.u32 %0, %%smid;" : "=r"(r.smid));
    r.kind = kind;
    r.t_entry = t0;
    r.t_ready = t1;
    r.t_aux = t2;
    r.t_exit = gtimer();
    g_trace.rec[i] = r;
  }
};
// an extra record with four phase marks of one CTA (kind TK_PHASE | ...), for kernels
// whose internal phases are being profiled
RT_DEV void trace_phase(uint32_t kind, unsigned long long a, unsigned long long b, unsigned long long c,
                        unsigned long long d) {
  if (!g_trace.rec) return;
  const unsigned i = atomicAdd(g_trace.n, 1u);
  if (i >= g_trace.cap) return;
  TraceRec r;
  asm volatile("mov.u64 %0, %%gridid;" : "=l"(r.grid));
  asm volatile("mov.u32 %0, %%smid;" : "=r"(r.smid));
  r.kind = kind;
  r.t_entry = a;
  r.t_ready = b;
  r.t_aux = c;
  r.t_exit = d;
  g_trace.rec[i] = r;
}
#define RT_TRACE_BINDER(fn)                                       \
  void fn(void* rec, unsigned* n, unsigned cap) {                 \
    TraceBuf b{reinterpret_cast<TraceRec*>(rec), n, cap};         \
    cudaMemcpyToSymbol(g_trace, &b, sizeof b);                    \
  }

// --------------------------------------------------------------- PTX wrappers
RT_DEV uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

RT_DEV void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
RT_DEV void fence_mbar_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
RT_DEV void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
// generic-proxy global writes before async-proxy (bulk copy) reads of the same bytes
RT_DEV void fence_proxy_async_global() { asm volatile("fence.proxy.async.global;" ::: "memory"); }
RT_DEV void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
RT_DEV void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
RT_DEV void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@P1 bra DONE_%=;\n\t"
      "bra WAIT_%=;\n\t"
      "DONE_%=:\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
// 1-D bulk async copy global -> shared (TMA engine, no tensor map): SASS UBLKCP
RT_DEV void bulk_g2s(void* smem_dst, const void* gmem_src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(smem_dst)),
      "l"(gmem_src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
// L2 eviction-priority policy for data read exactly once per step (decode weight tiles,
// decode KV pages): evict_first keeps the 126 MB L2 for what is re-read — kernel code
// (an epilogue's instructions are otherwise re-fetched from HBM every launch, since the
// L2 turns over every ~20 us under 6.5 TB/s of streaming), activations, page tables.
RT_DEV uint64_t l2_policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
// bulk_g2s with an L2 cache policy (policy 0 = no hint)
RT_DEV void bulk_g2s_hint(void* smem_dst, const void* gmem_src, uint32_t bytes, uint64_t* bar, uint64_t policy) {
  if (!policy) {
    bulk_g2s(smem_dst, gmem_src, bytes, bar);
    return;
  }
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          smem_u32(smem_dst)),
      "l"(gmem_src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}
RT_DEV void ldmatrix_x4(uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3, uint32_t addr) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}
RT_DEV void ldmatrix_x4_trans(uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3, uint32_t addr) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}
// D(16x8 f32) += A(16x16 bf16, row) * B(16x8 bf16, col)
RT_DEV void mma_bf16_16816(float* d, const uint32_t* a, const uint32_t* b) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
}

// ------------------------------------------------------- KV page swizzle
// A (page, kv head) block: [2 (K,V)][16 tok][hd] bf16; inside a 16 x hd matrix the
// 16-byte chunk c of token row j is stored at chunk c ^ ((j >> s) & m).
template <int HD>
struct KvSwz {
  static constexpr int CR = HD / 8;                 // 16B chunks per row
  static constexpr int M = (CR >= 8 ? 8 : CR) - 1;  // xor mask
  static constexpr int S = (CR >= 8 ? 0 : (CR == 4 ? 1 : 2));
  static constexpr int ROW_BYTES = HD * 2;
  static constexpr int MAT_BYTES = 16 * ROW_BYTES;  // one K or V matrix
  static constexpr int BLOCK_BYTES = 2 * MAT_BYTES; // K + V of one (page, head)
  RT_DEV static int chunk_off(int j, int c) { return j * ROW_BYTES + ((c ^ ((j >> S) & M)) << 4); }
  // byte offset of element (j, d) inside a K or V matrix
  RT_DEV static int elem_off(int j, int d) { return chunk_off(j, d >> 3) + ((d & 7) << 1); }
};

__host__ __device__ inline int kv_swz_chunk(int hd, int j, int c) {
  int cr = hd / 8;
  int m = (cr >= 8 ? 8 : cr) - 1;
  int s = (cr >= 8 ? 0 : (cr == 4 ? 1 : 2));
  return c ^ ((j >> s) & m);
}
